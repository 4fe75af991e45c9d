# A/B of solver-pass variants: bash tools/ab.sh "ENV1=..;ENV2=.." ...   (each arg one variant)
for v in "$@"; do
  echo "== $v"
  env $v python tools/probe.py ocean_1m 10 2>&1 | sed -n '4p;5p;$p'
done

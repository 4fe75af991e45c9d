for sc in 1.0 0.5 0.25 0.125; do echo "== $sc"; python tools/probe.py ocean_1m 10 $sc 2>&1 | sed -n '5p;$p'; done

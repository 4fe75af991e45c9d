# Per-launch times of selected kernels for library variants (cold, serialised;
# compare variants, not absolutes):
#   bash tools/ncu_kab.sh "<kernel regex>" libapbf_gpu.so libapbf_gpu_v0.so ...
re=$1; shift
for lib in "$@"; do
  echo "== $lib"
  APBF_LIB=$lib ncu --clock-control none --metrics gpu__time_duration.sum -k "regex:$re" --launch-skip 6 --launch-count 12 \
    python tools/probe.py ocean_1m 8 2>&1 | grep -E "^  [a-z_]+|gpu__time_duration" | paste - - | \
    awk '{n=$1; t[n]+=$NF; c[n]++} END {for (k in t) printf "%-28s %8.1f us  (%d launches)\n", k, t[k]/c[k], c[k]}'
done

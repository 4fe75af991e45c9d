# bench.py device-resident and e2e ms/step for library variants, alternating:
#   bash tools/bench_ab.sh libapbf_gpu.so libapbf_gpu_v0.so
for r in $(seq ${REPS:-2}); do for lib in "$@"; do
  APBF_LIB=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.load(sys.stdin); print('$lib', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3))"
done; done

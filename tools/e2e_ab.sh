# bench.py device and e2e ms/step of two library builds, alternated 3 times:
# bash tools/e2e_ab.sh libA.so libB.so
for r in 1 2 3; do for lib in "$@"; do APBF_LIB=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fast 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))"; done; done

# e2e ms/step with and without an environment setting, alternated 3 times:
# bash tools/e2e_env_ab.sh VAR=value
for r in 1 2 3; do for e in "" "$1"; do env $e python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fast 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e]', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))"; done; done

# A/B of library switches on the cfg4 bench: phase times per variant
run() { env "$@" timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items() if k in ('fwd_levels','bwd_levels')})"; }
run CAVS_PBWD=0
run CAVS_PBWD=1
run CAVS_PBWD=1 CAVS_PBWD_MAXNT=32
run CAVS_PBWD=1 CAVS_PBWD_MAXNT=16

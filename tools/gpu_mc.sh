mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "persistent or full_size_cfg4 or ksplit or cluster" > gpurun_out/pytest_mc.log 2>&1; echo mc tests rc=$?; tail -3 gpurun_out/pytest_mc.log | cut -c1-500
for MC in 1 0; do for C in cfg4 cfg3 cfg2; do
  CAVS_PERSIST_MC=$MC timeout 300 python bench.py --config $C --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('mc=$MC $C', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items() if k in ('fwd_levels','bwd_levels')})"
done; done

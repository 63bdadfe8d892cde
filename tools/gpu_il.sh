mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "persistent or full_size_cfg4 or bf16_parity" > gpurun_out/pytest_il.log 2>&1; echo il tests rc=$?; tail -3 gpurun_out/pytest_il.log | cut -c1-500
for IL in 4 1; do for C in cfg4 cfg3 cfg2; do
  CAVS_PERSIST_IL=$IL timeout 300 python bench.py --config $C --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('il=$IL $C', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items() if k in ('fwd_levels','bwd_levels')})"
done; done

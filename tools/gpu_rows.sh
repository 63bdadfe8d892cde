mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rows_level" > gpurun_out/pytest_rows.log 2>&1; echo rows rc=$?; tail -5 gpurun_out/pytest_rows.log | cut -c1-600
for C in cfg5 cfg4_h1024; do
  for PAIR in 1 0; do
    CAVS_ROWS_PAIR=$PAIR timeout 300 python bench.py --config $C --steps 10 --no-cpu-baseline --no-e2e 2>gpurun_out/b_$C_$PAIR.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$C pair=$PAIR', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items() if k in ('fwd_levels','bwd_levels')})"
  done
done

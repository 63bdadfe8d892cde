mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rows_level or cfg5 or persistent_levels" > gpurun_out/pytest_rows.log 2>&1; echo rows rc=$?; tail -3 gpurun_out/pytest_rows.log | cut -c1-600
for v in rows_pair rows_v8; do
 cp ab_libs/$v.so paper_1712_04048_b200/libcavs.so
 for C in cfg5 cfg4_h1024; do
  CAVS_ROWS_PAIR=0 timeout 300 python bench.py --config $C --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $C', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items() if k in ('fwd_levels','bwd_levels')})"
 done
done
cp ab_libs/rows_v8.so paper_1712_04048_b200/libcavs.so

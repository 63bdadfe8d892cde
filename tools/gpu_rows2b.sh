#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or full_size_cfg5" > gpurun_out/pytest_rows2b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rows2b.log
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), round(b['roofline']['frac'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})" || tail -3 gpurun_out/b.err
}
run cfg5 "X=1" "--config cfg5"
run cfg5_sel_items_lstm "CAVS_ROWS_SEL=i" "--config cfg4_h1024"
run cfg4_h1024 "X=1" "--config cfg4_h1024"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_rows --csv --log-file gpurun_out/rows2b.csv python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 --no-flush > /dev/null 2>&1; echo ncu rc=$?

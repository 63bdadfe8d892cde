#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or full_size_cfg5" > gpurun_out/pytest_dsm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dsm.log; grep -E "^FAILED|Error" gpurun_out/pytest_dsm.log | head -5
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graph 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), round(b['roofline']['frac'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})" || tail -3 gpurun_out/b.err
}
run cfg5 "X=1" "--config cfg5"
run cfg5_global "CAVS_ROWS_DSM=0" "--config cfg5"
TRACE_ITERS=3 timeout 300 python tools/trace_rows.py cfg5 > gpurun_out/trace_rows_cfg5_dsm.txt 2>&1; tail -20 gpurun_out/trace_rows_cfg5_dsm.txt

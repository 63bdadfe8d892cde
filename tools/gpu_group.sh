#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})" || tail -3 gpurun_out/b.err
}
run h1024 "X=1" "--config cfg4_h1024"
run h1024_legacy "CAVS_TC_GROUP=0" "--config cfg4_h1024"
run fp32 "X=1" "--config cfg4 --precision fp32"
run fp32_legacy "CAVS_TC_GROUP=0" "--config cfg4 --precision fp32"
run cfg5 "X=1" "--config cfg5"
run cfg4 "X=1" "--config cfg4"

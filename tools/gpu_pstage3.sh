#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), 'eager', round(b['eager']['value']), 'e2e', b['e2e']['value'] if b.get('e2e') else None, {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if 'levels' in k})" || tail -3 gpurun_out/b.err
}
run cfg4 "X=1" "--config cfg4"
run cfg3 "X=1" "--config cfg3"
run cfg2 "X=1" "--config cfg2"
run cfg4_inf "X=1" "--config cfg4 --inference"
run cfg4_fc512 "X=1" "--config cfg5 --h 512"

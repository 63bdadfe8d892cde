#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "ksliced or gate_split or tcgen05 or fp32_tensor or full_size_cfg4" > gpurun_out/pytest_ksl.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|Error:" gpurun_out/pytest_ksl.log | tail -12
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), round(b['roofline']['frac'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})" || tail -3 gpurun_out/b.err
}
run cfg4_fp32 "X=1" "--config cfg4 --precision fp32"
run cfg4_fp32_ksl1 "CAVS_TC_KSL=1" "--config cfg4 --precision fp32"
run cfg4_fp32_ksl2 "CAVS_TC_KSL=2" "--config cfg4 --precision fp32"
run cfg4_h1024 "X=1" "--config cfg4_h1024"
run cfg4_h1024_ksl1 "CAVS_TC_KSL=1" "--config cfg4_h1024"
run cfg4_h1024_ksl2 "CAVS_TC_KSL=2" "--config cfg4_h1024"
run cfg5 "X=1" "--config cfg5"

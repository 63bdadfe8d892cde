#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "bf16_parity or full_size_cfg4 or persistent_levels or dx_records or shared_pull or lazy or dag_parity" > gpurun_out/pytest_dx.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dx.log; grep -E "^FAILED" gpurun_out/pytest_dx.log | head
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if k in ('dx','lazy','xproj')})" || tail -3 gpurun_out/b.err
}
run cfg4 "X=1" "--config cfg4"
run cfg4_kpb1 "CAVS_DX_KPB=1" "--config cfg4"
run cfg3 "X=1" "--config cfg3"
run h1024 "X=1" "--config cfg4_h1024"
run h1024_kpb1 "CAVS_DX_KPB=1" "--config cfg4_h1024"

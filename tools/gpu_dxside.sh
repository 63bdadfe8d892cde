#!/bin/bash
# r02: dX on the side stream beside the lazy weight-gradient GEMMs (CAVS_DX_SIDE=1 default) vs main stream
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "full_size or dx or graph or sync_free or rows_xproj or persistent_levels or dag or fp32" > gpurun_out/pytest_dxside.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dxside.log; grep -E "^FAILED" gpurun_out/pytest_dxside.log | head -8
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 30 --warmup 5 --no-cpu-baseline 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), 'e2e', round(b['e2e']['value']), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if k in ('lazy','dx','reduce')})" || tail -3 gpurun_out/b.err
}
for r in 1 2; do for c in cfg4 cfg3 cfg5 cfg4_h1024; do
  run "${c}_dxside0" "CAVS_DX_SIDE=0" "--config $c"
  run "${c}_dxside1" "CAVS_DX_SIDE=1" "--config $c"
done; done

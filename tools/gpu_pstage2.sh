#!/bin/bash
mkdir -p gpurun_out
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), 'eager', round(b['eager']['value']), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if 'levels' in k})" || tail -3 gpurun_out/b.err
}
run cfg4_nanosleep "X=1" "--config cfg4"
run cfg4_bwd80k "CAVS_PERSIST_STAGE_BWD=81920" "--config cfg4"
run cfg4_bwd64k "CAVS_PERSIST_STAGE_BWD=65536" "--config cfg4"
run cfg4_fwd64k "CAVS_PERSIST_STAGE_FWD=65536" "--config cfg4"
run cfg3 "X=1" "--config cfg3"
run cfg3_bwd80k "CAVS_PERSIST_STAGE_BWD=81920" "--config cfg3"
CAVS_PERSIST_STAGE_BWD=81920 timeout 300 python tools/trace_persist.py cfg4 > gpurun_out/trace_persist_b80.txt 2>&1; grep -A14 "MMA kind 4002" gpurun_out/trace_persist_b80.txt | head -16; grep -A8 "MMA kind 4000" gpurun_out/trace_persist_b80.txt | head -10

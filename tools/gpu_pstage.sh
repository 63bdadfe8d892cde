#!/bin/bash
mkdir -p gpurun_out
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), 'eager', round(b['eager']['value']), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if 'levels' in k})" || tail -3 gpurun_out/b.err
}
run cfg4 "X=1" "--config cfg4"
run cfg4_st16 "CAVS_PERSIST_STAGE=16384" "--config cfg4"
run cfg4_st32 "CAVS_PERSIST_STAGE=32768" "--config cfg4"
run cfg4_st16_mc "CAVS_PERSIST_STAGE=16384 CAVS_PERSIST_MC=1" "--config cfg4"
run cfg3 "X=1" "--config cfg3"
run cfg3_st16 "CAVS_PERSIST_STAGE=16384" "--config cfg3"
CAVS_PERSIST_STAGE=16384 timeout 300 python tools/trace_persist.py cfg4 > gpurun_out/trace_persist_st16.txt 2>&1; grep -A14 "MMA kind 4002" gpurun_out/trace_persist_st16.txt | head -16

#!/bin/bash
# r02: persistent-kernel B stage sweep on the N = 1 chain configs (cfg3 Var-LSTM, cfg2 Fixed-LSTM)
mkdir -p gpurun_out
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items() if 'levels' in k}, b['config']['engine'][:160])" || tail -3 gpurun_out/b.err
}
for c in cfg3 cfg2; do
  run ${c}_default "X=1" "--config $c"
  for v in 32768 49152 65536 81920 98304; do run ${c}_bwd$v "CAVS_PERSIST_STAGE_BWD=$v" "--config $c"; done
  for v in 32768 65536 98304; do run ${c}_fwd$v "CAVS_PERSIST_STAGE_FWD=$v" "--config $c"; done
done

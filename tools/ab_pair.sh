#!/bin/bash
mkdir -p gpurun_out
for C in cfg5 cfg4_h1024; do for P in 0 1; do
  CAVS_ROWS_PAIR=$P timeout 300 python bench.py --config $C --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-graph 2>/dev/null | tail -1 > gpurun_out/ab_pair_${C}_$P.json
  python -c "
import json; b=json.load(open('gpurun_out/ab_pair_${C}_$P.json')); print('$C pair=$P', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})"
done; done

#!/bin/bash
mkdir -p gpurun_out
run() {  # name env args
  env $2 timeout 300 python bench.py $3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | tail -1 > gpurun_out/b.json
  python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('$1', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})" || tail -3 gpurun_out/b.err
}
run h1024 "X=1" "--config cfg4_h1024"
run h1024_skinny0 "CAVS_SKINNY_MAX=0" "--config cfg4_h1024"
run h1024_skinny4 "CAVS_SKINNY_MAX=4" "--config cfg4_h1024"
run h1024_ksl4 "CAVS_TC_KSL=4" "--config cfg4_h1024"
run h1024_skinny0_ksl4 "CAVS_SKINNY_MAX=0 CAVS_TC_KSL=4" "--config cfg4_h1024"
run cfg5_skinny0 "CAVS_SKINNY_MAX=0" "--config cfg5"

#!/bin/bash
# A/B of prebuilt libraries (ab_libs/<name>.so) on the GPU box: VARIANTS="a b" CONFIGS="cfg4 cfg3" bash tools/ab_libs.sh
mkdir -p gpurun_out
run() {
  cp ab_libs/$1.so paper_1712_04048_b200/libcavs.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 3 --config $2 ${BENCH_ARGS} 2>&1 | tail -1 > gpurun_out/b_$1_$2.json
  python -c "
import json; b=json.load(open('gpurun_out/b_$1_$2.json')); print('$1 $2', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})"
}
for c in ${CONFIGS:-cfg4}; do for v in ${VARIANTS}; do run $v $c; done; done

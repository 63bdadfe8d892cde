#!/bin/bash
# ncu --set full of one kernel (regex $K) of a short bench run, plus the bench phases.
# usage (GPU box): K=k_lazy [S=2] [C=1] [BENCH_ARGS=...] bash tools/prof_kernel.sh
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null > gpurun_out/bench_k.json
python -c "
import json; b=json.loads(open('gpurun_out/bench_k.json').read().strip().splitlines()[-1]); print(round(b['value']), round(b['ms_per_step'],4))
for k,v in b['phases'].items(): print(k, round(v['ms_per_step'],4), v['TFLOP/s'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${K}" -s ${S:-2} -c ${C:-1} \
    -o gpurun_out/${OUT:-kernel} -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 ${BENCH_ARGS} \
    > gpurun_out/${OUT:-kernel}.log 2>&1
tail -2 gpurun_out/${OUT:-kernel}.log

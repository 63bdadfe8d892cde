#!/bin/bash
# Run on the GPU box (gpurun): launch list + full capture of the level kernels.
set -x
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 ${BENCH_ARGS}"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_typeI -s ${SKIP:-1} -c ${COUNT:-6} \
    -o gpurun_out/prof_levels -f python bench.py $ARGS > gpurun_out/prof_levels.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_typeII -c 3 \
    -o gpurun_out/prof_lazy -f python bench.py $ARGS > gpurun_out/prof_lazy.log 2>&1
ls -la gpurun_out

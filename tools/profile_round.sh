#!/bin/bash
# Round profile capture (run on the GPU box via gpurun).  Produces, under gpurun_out/:
#   launches.csv      ncu launch list (gpu__time_duration.sum, --clock-control none) of the bench command
#   levels.ncu-rep    ncu --set full of one forward+backward pass worth of level kernels (warm caches)
#   bench.json        the bench line of the same command (no profiler attached)
set -x
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 ${BENCH_ARGS}"
python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_tc_level|k_skinny|k_tc_typeII" -s ${SKIP:-60} -c ${COUNT:-60} \
    -o gpurun_out/levels -f python bench.py $ARGS > gpurun_out/levels.log 2>&1
ls -la gpurun_out

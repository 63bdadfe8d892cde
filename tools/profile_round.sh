#!/bin/bash
# Round capture (run on the GPU box via gpurun).  Produces, under gpurun_out/:
#   pytest_gpu.log    the -m gpu parity suite
#   bench.json        the bench line (no profiler attached)
#   launches.csv      ncu launch list (gpu__time_duration.sum, --clock-control none) of a short bench
#   persist.ncu-rep   ncu --set full of the persistent level kernels (one forward + one backward pass)
#   rows.ncu-rep      ncu --set full of the row GEMMs and the lazy (type-II) GEMMs
set -x
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 ${BENCH_ARGS}"
if [ -z "${SKIP_TESTS}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_persist" -s ${SKIP:-2} -c ${COUNT:-2} \
    -o gpurun_out/persist -f python bench.py $ARGS > gpurun_out/persist.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_gemm_rows|k_lazy|k_graph_sched|k_level_offsets|k_build_maps|k_colsum" -s 6 -c 7 \
    -o gpurun_out/rows -f python bench.py $ARGS > gpurun_out/rows.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_rows|k_lazy" -s 0 -c 3 \
    -o gpurun_out/cfg5 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 --config cfg5 > gpurun_out/cfg5.log 2>&1
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
ls -la gpurun_out

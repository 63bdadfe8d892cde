#!/bin/bash
# r02: k_prep with 4 loads in flight per thread (plain copies) and two tiles per pass (transposes)
mkdir -p gpurun_out
cp ab_libs/prep4.so paper_1712_04048_b200/libcavs.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "full_size or fp32 or bf16_parity or rows_xproj or persistent_levels" > gpurun_out/pytest_prep.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_prep.log; grep -E "^FAILED" gpurun_out/pytest_prep.log | head -8
VARIANTS="head prep4" CONFIGS="cfg5 cfg4 cfg4_h1024" bash tools/ab_libs.sh
BENCH_ARGS="--precision fp32" VARIANTS="head prep4" CONFIGS="cfg4" bash tools/ab_libs.sh
VARIANTS="head prep4" CONFIGS="cfg5 cfg4" bash tools/ab_libs.sh
cp ab_libs/prep4.so paper_1712_04048_b200/libcavs.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prep|k_pull" -c 4 --csv --log-file gpurun_out/launches_prep_cfg5.csv \
    python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --pool 2 > gpurun_out/launches_prep.log 2>&1; echo "launch list rc=$?"

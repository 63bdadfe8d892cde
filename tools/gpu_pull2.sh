#!/bin/bash
# r02: k_pull 512 threads for grids of <= 2 tiles per SM; cfg5 launch list (prep vs pull)
mkdir -p gpurun_out
cp ab_libs/pull512.so paper_1712_04048_b200/libcavs.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "pull or dx or xrow or x_row or full_size_cfg4 or full_size_cfg5 or dag" > gpurun_out/pytest_pull.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pull.log; grep -E "^FAILED" gpurun_out/pytest_pull.log | head -8
VARIANTS="head pull512" CONFIGS="cfg4 cfg5 cfg3" bash tools/ab_libs.sh
VARIANTS="head pull512" CONFIGS="cfg4 cfg5" bash tools/ab_libs.sh
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg5.csv \
    python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --pool 2 > gpurun_out/launches_cfg5.log 2>&1; echo "launch list rc=$?"

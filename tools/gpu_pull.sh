#!/bin/bash
# r02: k_pull with 512 threads per 64-row tile (pull512) vs 256 (head)
mkdir -p gpurun_out
cp ab_libs/pull512.so paper_1712_04048_b200/libcavs.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "pull or dx or xrow or x_row or full_size_cfg4 or full_size_cfg5 or fp32_tensor or dag" > gpurun_out/pytest_pull.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pull.log; grep -E "^FAILED" gpurun_out/pytest_pull.log | head -8
VARIANTS="head pull512" CONFIGS="cfg4 cfg3 cfg5" bash tools/ab_libs.sh
VARIANTS="head pull512" CONFIGS="cfg4 cfg5" bash tools/ab_libs.sh

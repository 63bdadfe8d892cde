#!/bin/bash
# r02: one 4-D TMA box per B stage in k_rows (b4) vs the previous multi-box stages
mkdir -p gpurun_out
cp ab_libs/b4.so paper_1712_04048_b200/libcavs.so
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "rows or full_size_cfg5 or persistent_levels or full_size_sampled or ksliced" > gpurun_out/pytest_b4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_b4.log; grep -E "^FAILED" gpurun_out/pytest_b4.log | head -8
VARIANTS="base b4" CONFIGS="cfg5 cfg4_h1024 cfg2" bash tools/ab_libs.sh
CAVS_ROWS_XD=1 VARIANTS="base b4" CONFIGS="cfg4" bash tools/ab_libs.sh
VARIANTS="base b4" CONFIGS="cfg5 cfg4_h1024" bash tools/ab_libs.sh

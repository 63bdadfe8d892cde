#!/bin/bash
# r02: dx zeroing on the side stream with dX; dZ tail-row zeroing beside the pull (dxz) vs before (dxs)
mkdir -p gpurun_out
cp ab_libs/dxz.so paper_1712_04048_b200/libcavs.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_dxz.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dxz.log; grep -E "^FAILED" gpurun_out/pytest_dxz.log | head -8
VARIANTS="dxs dxz" CONFIGS="cfg4 cfg3 cfg2" bash tools/ab_libs.sh
VARIANTS="dxs dxz" CONFIGS="cfg4 cfg3" bash tools/ab_libs.sh
cp ab_libs/dxz.so paper_1712_04048_b200/libcavs.so

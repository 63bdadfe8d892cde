#!/bin/bash
# r02: PDL launch_dependents at the start of the persistent kernels (ptrig) vs head
mkdir -p gpurun_out
cp ab_libs/ptrig.so paper_1712_04048_b200/libcavs.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_ptrig.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ptrig.log; grep -E "^FAILED" gpurun_out/pytest_ptrig.log | head -8
VARIANTS="head ptrig" CONFIGS="cfg4 cfg3 cfg2" bash tools/ab_libs.sh
VARIANTS="head ptrig" CONFIGS="cfg4 cfg3" bash tools/ab_libs.sh
cp ab_libs/ptrig.so paper_1712_04048_b200/libcavs.so

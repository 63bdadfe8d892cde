#!/bin/bash
# r02: PDL launch_dependents in the x-projection / dX row GEMM and k_roots (trig) vs implicit trigger at exit (head)
mkdir -p gpurun_out
cp ab_libs/trig.so paper_1712_04048_b200/libcavs.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_trig.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_trig.log; grep -E "^FAILED" gpurun_out/pytest_trig.log | head -8
VARIANTS="head trig" CONFIGS="cfg4 cfg3 cfg2 cfg4_h1024" bash tools/ab_libs.sh
VARIANTS="head trig" CONFIGS="cfg4 cfg3" bash tools/ab_libs.sh
cp ab_libs/trig.so paper_1712_04048_b200/libcavs.so

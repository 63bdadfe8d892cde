#!/bin/bash
# r02: PDL triggers in k_graph_sched, k_level_offsets, k_pull (strig) vs head
mkdir -p gpurun_out
cp ab_libs/strig.so paper_1712_04048_b200/libcavs.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_strig.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_strig.log; grep -E "^FAILED" gpurun_out/pytest_strig.log | head -8
VARIANTS="head strig" CONFIGS="cfg4 cfg3 cfg2" bash tools/ab_libs.sh
VARIANTS="head strig" CONFIGS="cfg4 cfg3" bash tools/ab_libs.sh
cp ab_libs/strig.so paper_1712_04048_b200/libcavs.so

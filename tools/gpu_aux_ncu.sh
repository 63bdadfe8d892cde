#!/bin/bash
# r02 (end): ncu --set full of the cfg4 non-level kernels (lazy, x-projection / dX row GEMMs, db) -> gpurun_out/aux_*.csv
mkdir -p gpurun_out
for K in k_lazy k_gemm_rows k_colsum; do
  timeout 600 ncu --set full --clock-control none -k regex:"$K" -s 2 -c 2 --csv --page raw \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/aux_$K.csv 2> gpurun_out/aux_$K.err
  echo "$K rc=$?"
done

#!/bin/bash
# ncu --set full of the row-tiled level kernels (k_rows) at cfg5 (Tree-FC h=2048) and cfg4 h=1024.
mkdir -p gpurun_out
for C in cfg5 cfg4_h1024; do
  timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows" -s 0 -c 4 \
    -o gpurun_out/rows_$C -f python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 \
    > gpurun_out/rows_$C.log 2>&1; echo "$C rc=$?"
done

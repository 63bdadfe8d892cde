#!/bin/bash
# ncu --set full of the first k_rows launch at cfg5 (Tree-FC h=2048, forward level 1: 8192 rows),
# single CTA vs CTA pairs (CAVS_ROWS_PAIR=1) -> gpurun_out/rows_l1_p{0,1}.ncu-rep
mkdir -p gpurun_out
for P in 0 1; do
  CAVS_ROWS_PAIR=$P timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows" -s 0 -c 1 \
    -o gpurun_out/rows_l1_p$P -f python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 --no-graph \
    > gpurun_out/rows_l1_p$P.log 2>&1; echo "pair=$P rc=$?"
done

#!/bin/bash
# ncu --set full of small cfg5 level launches of k_rows (split-K shares): forward levels 6 and 8
mkdir -p gpurun_out
for S in 5 7; do
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows" -s $S -c 1 \
    -o gpurun_out/rows_small_s$S -f python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 --no-graph \
    > gpurun_out/rows_small_s$S.log 2>&1; echo "s=$S rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or lazy or full_size_cfg4 or dag_parity or sync_free or async" > gpurun_out/pytest_dbside.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dbside.log
for E in 1 0; do CAVS_DB_SIDE=$E timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b.json
python -c "
import json; b=json.load(open('gpurun_out/b.json')); print('cfg4 db_side=$E', round(b['value']), round(b['ms_per_step'],4), round(b['eager']['value']), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})"; done

#!/bin/bash
# Tensor-pipe utilisation of every kernel of one training step (ncu metrics pass, no replay of
# the whole section set): CONFIG=cfg4_h1024 bash tools/prof_tensor_pipe.sh -> gpurun_out/tp_<config>.csv
mkdir -p gpurun_out
C=${CONFIG:-cfg4_h1024}
timeout 300 python bench.py --config $C --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/bench_$C.json
python -c "
import json; b=json.loads(open('gpurun_out/bench_$C.json').read().strip().splitlines()[-1]); print('$C', round(b['value']), round(b['ms_per_step'],4))
for k,v in b['phases'].items(): print('  ', k, round(v['ms_per_step'],4), v['TFLOP/s'])"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  --clock-control none --csv --log-file gpurun_out/tp_$C.csv \
  python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 --no-flush > gpurun_out/tp_$C.log 2>&1
echo ncu rc=$?

#!/bin/bash
# Final round-2 evidence on one B200 -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['kernel'],d['roofline']['frac'],d['cpu_baseline']['value'],d['clocks'])"
for C in "cfg1" "cfg2" "cfg3" "cfg4_h1024" "cfg5" "cfg4 --precision fp32" "cfg4 --inference"; do
  N=$(echo $C | tr ' ' '_' | tr -d '-')
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$N.json 2> gpurun_out/cfg_$N.err
  python -c "import json;d=json.loads(open('gpurun_out/cfg_$N.json').read().strip().splitlines()[-1]);print('$N',round(d['value']),round(d['ms_per_step'],4),d['e2e']['value'] if d.get('e2e') else None,d['roofline']['kernel'],round(d['roofline']['frac'],4))" || tail -3 gpurun_out/cfg_$N.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_persist" -s 2 -c 2 \
    -o gpurun_out/persist -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/persist.log 2>&1; echo "ncu full rc=$?"
for C in cfg5 cfg4_h1024; do CONFIG=$C bash tools/prof_tensor_pipe.sh > /dev/null 2>&1; python tools/tp_summary.py gpurun_out/tp_$C.csv > gpurun_out/tp_$C.txt; tail -1 gpurun_out/tp_$C.txt; done

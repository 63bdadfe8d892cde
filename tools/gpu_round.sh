#!/bin/bash
# Round evidence on one B200: the -m gpu suite, smoke, the default bench line, the ncu launch list
# of a short bench, ncu --set full of the top kernel (persistent backward) -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['kernel'],d['roofline']['frac'],d['cpu_baseline']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_persist" -s 2 -c 2 \
    -o gpurun_out/persist -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/persist.log 2>&1; echo "ncu full rc=$?"

mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ksplit or persistent or benchmark_shape" > gpurun_out/pytest_ksplit.log 2>&1; echo ksplit rc=$?; tail -25 gpurun_out/pytest_ksplit.log | cut -c1-800
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ks.json 2> gpurun_out/bench_ks.err; echo bench rc=$?; tail -c 300 gpurun_out/bench_ks.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_ks.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"])
print({k: round(v["ms_per_step"]*1000,1) for k,v in d["phases"].items()})
PY
CAVS_PBWD=0 timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ks0.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_ks0.json').read().strip().splitlines()[-1]);print('old', d['value'], {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items()})"

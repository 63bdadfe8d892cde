# end-of-round bench lines of every BASELINE config (1 x B200) + the LM step -> gpurun_out/
mkdir -p gpurun_out
for C in cfg1 cfg2 cfg3 cfg4 cfg4_h1024 cfg5; do
  timeout 400 python bench.py --config $C --steps 20 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$C.json').read().strip().splitlines()[-1])
g=d.get('graph') or {}; e=d.get('eager') or {}
print('$C', d['dtype'], round(d['value']), round(d['ms_per_step'],4), 'eager', round(e.get('value',0)), 'e2e', round((d.get('e2e') or {}).get('value',0)), 'frac', round(d['roofline']['frac'],4))"
done
timeout 300 python bench.py --config cfg4 --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_fp32.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg4_fp32.json').read().strip().splitlines()[-1]); print('cfg4 fp32', round(d['value']), round(d['ms_per_step'],3))"
timeout 300 python bench.py --config cfg4 --inference --steps 20 --no-cpu-baseline > gpurun_out/bench_cfg4_inf.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg4_inf.json').read().strip().splitlines()[-1]); print('cfg4 inference', round(d['value']), round(d['ms_per_step'],4))"
timeout 300 python tools/bench_lm.py > gpurun_out/bench_lm.json 2> gpurun_out/bench_lm.err; tail -c 600 gpurun_out/bench_lm.json; tail -3 gpurun_out/bench_lm.err

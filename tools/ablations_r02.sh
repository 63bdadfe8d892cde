#!/bin/bash
# Round-2 ablations on one B200 (Fig. 10 / §5.3): the
# paper's own optimisation axes as library toggles, on the per-task engine they apply to, plus
# Fig. 10's batched-vs-serial curve on Fixed-LSTM.  Output: gpurun_out/ablations_r02.jsonl
mkdir -p gpurun_out
OUT=gpurun_out/ablations_r02.jsonl
: > $OUT
run() {
  local cfg="$1" name="$2"; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 --warmup 3 ${BENCH_ARGS} 2>/dev/null | tail -1 | \
    python -c "import json,sys; b=json.loads(sys.stdin.read()); print(json.dumps({'config': '$cfg', 'variant': '$name', 'precision': b['dtype'], 'samples_per_s': round(b['value'],1), 'ms_per_step': round(b['ms_per_step'],4), 'phases': {k: round(v['ms_per_step'], 4) for k, v in b['phases'].items()}}))" >> $OUT
  tail -1 $OUT | cut -c1-200
}
for cfg in cfg4 cfg3; do
  run $cfg "default engine (persistent level kernels)"
  run $cfg "per-task launches (baseline of the toggles below)" CAVS_PERSIST=0
  run $cfg "per-task + lazy batching OFF" CAVS_PERSIST=0 CAVS_LAZY_BATCH=0
  run $cfg "per-task + unfused cell epilogues" CAVS_UNFUSED=1
  run $cfg "per-task + streamed x-projection" CAVS_STREAMING=1
  run $cfg "per-task + all three off" CAVS_LAZY_BATCH=0 CAVS_UNFUSED=1
done
BENCH_ARGS="--precision fp32" run cfg4 "fp32 default"
BENCH_ARGS="--precision fp32" run cfg4 "fp32 lazy batching OFF" CAVS_LAZY_BATCH=0
BENCH_ARGS="--precision fp32" run cfg4 "fp32 unfused" CAVS_UNFUSED=1
timeout 1200 python tools/serial_vs_batched.py --config cfg2 --sweep 2,4,8,16,32,64,128 --reps 3 >> $OUT 2>gpurun_out/svb.err
tail -7 $OUT

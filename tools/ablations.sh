#!/bin/bash
# Engine ablations on one B200 (the structure of PAPER.md Fig. 10): each
# toggle switches one design choice off; same cfg4 workload, bench.py device time.
mkdir -p gpurun_out
OUT=gpurun_out/ablations.jsonl
: > $OUT
run() {
  local name="$1"; shift
  env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 ${BENCH_ARGS} 2>/dev/null | tail -1 | \
    python -c "import json,sys; b=json.loads(sys.stdin.read()); print(json.dumps({'variant': '$name', 'samples_per_s': b['value'], 'ms_per_step': b['ms_per_step'], 'phases': {k: round(v['ms_per_step'], 4) for k, v in b['phases'].items()}}))" >> $OUT
  tail -1 $OUT | cut -c1-160
}
run "all on (default)"
run "per-task level launches (no persistent kernel)" CAVS_PERSIST=0
run "per-task launches, monolithic CTAs (no gate-split clusters)" CAVS_PERSIST=0 CAVS_TC_MONO=1
run "split-K lazy GEMMs + pack (no stream-K)" CAVS_LAZY=0
run "x-projection / dX on per-task kernels (no row GEMMs)" CAVS_GEMM_ROWS=0
run "FFMA instead of tensor cores (bf16 operands)" CAVS_BF16_SIMT=1
BENCH_ARGS="--precision fp32" run "fp32 mode (FFMA, fp32 operands)"
timeout 900 python tools/serial_vs_batched.py >> $OUT 2>/dev/null; tail -1 $OUT

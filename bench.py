#!/usr/bin/env python
"""Benchmark of the Cavs level-batched F-over-G training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cavs|reference]
                    [--config cfg4] [--precision bf16|fp32] [--h H]

Workload (BASELINE.json metric "Tree-LSTM train samples/s (fwd+bwd)"): cfg4 = Tree-LSTM on
synthetic SST-shaped binarised parse trees, h = d = 512, a GLOBAL batch of 256 trees (strong
scaling: at N > 1 the batch is sharded over the ranks by vertex count, dp.shard_batch; --weak
gives every rank its own 256 trees).  A step = cavs_load_graphs (device-resident CSR) +
cavs_schedule + cavs_forward + cavs_backward (+ the bucketed NCCL all-reduce of the weight
gradients for N > 1, overlapped with dX / db) over one batch of a pool of 16 pre-generated
batches, so the schedule changes every step.  L2 is flushed (256 MiB write) between timed steps,
outside the per-step CUDA events.

The roofline object is computed live from the library's per-phase CUDA events and its
algorithmic FLOP counts; `traffic` comes from the
committed ncu capture in profiles/.  `cpu_baseline` / `--impl reference` time the fp64
CPU oracle (oracle/) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH_DESC = {
    "cfg1": "Tree-FC, 4 random binary trees of 8 leaves, hidden 16",
    "cfg2": "Fixed-LSTM LM, PTB-shaped synthetic tokens, seq len 64, hidden 512, batch 64",
    "cfg3": "Var-LSTM, SST-shaped lengths 1-56, hidden 512, batch 256",
    "cfg4": "Tree-LSTM, synthetic SST-shaped binarised parse trees, hidden 512, batch 256",
    "cfg4_h1024": "Tree-LSTM, synthetic SST-shaped binarised parse trees, hidden 1024, batch 256",
    "cfg5": "Tree-FC, complete binary trees of 256 leaves, hidden 2048, batch 64",
}
def _desc(cfg, h):
    """Workload description with the hidden size actually run (--h overrides the config's)."""
    import re
    return re.sub(r"hidden \d+", f"hidden {h}", BATCH_DESC.get(cfg, ""))


TENSOR_PHASES = ("xproj", "fwd_levels", "bwd_levels", "lazy", "dx")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cavs", choices=["cavs", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--precision", default=None, choices=["bf16", "fp32"],
                    help="default bf16; fp32 for cfg1 (BASELINE: 'hidden 16, fp32'; bf16 mode needs h % 64 == 0)")
    ap.add_argument("--h", type=int, default=None)
    ap.add_argument("--pool", type=int, default=16)
    ap.add_argument("--cpu-sample", type=int, default=48, help="graphs in the CPU-oracle baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: an independent batch of the config's size per rank (default: strong "
                         "scaling, ONE global batch sharded over the ranks by dp.shard_batch)")
    ap.add_argument("--no-graph", action="store_true",
                    help="skip the CUDA-graph measurement (sync-free mode: one captured graph per pool batch)")
    ap.add_argument("--inference", action="store_true",
                    help="forward-only (cavs_forward_inference): inference samples/s, no backward")
    a = ap.parse_args()
    if a.precision is None:
        a.precision = "fp32" if a.config == "cfg1" else "bf16"
    return a


# ------------------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------ CPU oracle
def _oracle_worker(args):
    import oracle
    from workloads import gen
    cell, N, h, d, params, gp, cp, ci, x_row, x, gamma = args
    b = gen.Batch(cell=cell, N=N, h=h, d=d, graph_ptr=gp, child_ptr=cp, child_idx=ci, x_row=x_row, x=x,
                  params=params, gamma=gamma)
    t = time.perf_counter()
    oracle.run(b)
    return time.perf_counter() - t


def _noop(_):
    return os.getpid()


def _oracle_jobs(b, graphs, n_chunks):
    from workloads import gen              # never the product package: the oracle leg must not load libcavs.so
    chunks = [graphs[i::n_chunks] for i in range(n_chunks)]
    jobs = []
    for ch in chunks:
        if not ch:
            continue
        gp, cp, ci, rows, recs, nxr = gen.subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, ch)
        jobs.append((b.cell, b.N, b.h, b.d, b.params, gp, cp, ci, nxr, b.x[recs], b.gamma[rows]))
    return jobs


class OraclePool:
    def __init__(self):
        import multiprocessing as mp
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        os.environ.setdefault("MKL_NUM_THREADS", "1")
        self.cores = len(os.sched_getaffinity(0))
        self.pool = mp.get_context("spawn").Pool(self.cores)
        self.pool.map(_noop, range(self.cores))           # start-up outside any timing

    def run(self, b, graphs):
        jobs = _oracle_jobs(b, graphs, min(self.cores, len(graphs)))
        t = time.perf_counter()
        cpu = sum(self.pool.map(_oracle_worker, jobs))
        return time.perf_counter() - t, cpu, len(jobs)

    def close(self):
        self.pool.terminate()


def cpu_baseline(args, unit_batch):
    from workloads import gen
    b = gen.make_config_batch(args.config, seed=0, h=args.h)
    n = min(args.cpu_sample, b.K)
    pool = OraclePool()
    wall, cpu, used = pool.run(b, list(range(n)))
    pool.close()
    n1 = min(4, b.K)                                  # one core, one process
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):                        # BLAS of this process on one thread
        one = _oracle_worker(_oracle_jobs(b, list(range(n1)), 1)[0])
    return {"value": n / wall, "unit": "samples/s", "cores": used, "kind": "oracle",
            "sample": f"{n} of the {b.K} graphs of batch seed 0 ({args.config}, h={b.h}), fp64 NumPy per-vertex "
                      f"evaluator, fwd+bwd, graphs split over {used} worker processes (1 thread each); "
                      f"{cpu:.1f} CPU-s in {wall:.2f} s wall",
            "one_core": {"value": n1 / one, "unit": "samples/s", "sample": f"graphs 0..{n1 - 1}, one process"}}


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    from workloads import gen
    b = gen.make_config_batch(args.config, seed=0, h=args.h)
    per_step = min(16, b.K)
    pool = OraclePool()
    times = []
    for i in range(args.warmup + args.steps):
        graphs = [(i * per_step + j) % b.K for j in range(per_step)]
        wall, cpu, used = pool.run(b, graphs)
        if i >= args.warmup:
            times.append(wall)
    pool.close()
    ms = 1000 * sum(times) / len(times)
    value = per_step / (ms / 1000)
    line = {
        "impl": "reference", "metric": "Tree-LSTM train samples/s (fwd+bwd)" if b.cell == "tree_lstm"
        else "Tree-FC train samples/s (fwd+bwd)",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config}: {_desc(args.config, b.h)}",
                                        "h": b.h, "batch": b.K, "sample_graphs_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": used, "kind": "oracle",
                         "sample": f"{per_step} graphs of {args.config} batch seed 0 per step"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1712_04048_b200 import Context, dp
    from workloads import gen

    # CAVS_DIST_BACKEND=gloo (test only): several ranks may then share one GPU (NCCL refuses that),
    # which exercises the sharded / bucketed data-parallel path on a single-GPU box
    backend = os.environ.get("CAVS_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # ---- inputs: a pool of batches resident in HBM before the timed region ----
    # strong scaling (default): pool batch i is ONE global batch (seed i, same on every rank), sharded
    # over the ranks by vertex count (dp.shard_batch; the graphs are independent);
    # weak scaling (--weak): every rank draws its own full-size batches (seeds rank * pool + i)
    if args.weak or world == 1:
        glob = [gen.make_config_batch(args.config, seed=(rank if args.weak else 0) * args.pool + i, h=args.h)
                for i in range(args.pool)]
        batches = glob
    else:
        glob = [gen.make_config_batch(args.config, seed=i, h=args.h) for i in range(args.pool)]
        batches = [dp.shard_batch(g, world, rank)[0] for g in glob]
    depth_T = float(np.mean([max(dp.graph_depths(g.graph_ptr, g.child_ptr, g.child_idx)) for g in glob]))
    b0 = batches[0]
    params = torch.from_numpy(gen.make_config_batch(args.config, seed=0, h=args.h).params).to(dev)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pool = [dict(gp=t(b.graph_ptr), cp=t(b.child_ptr), ci=t(b.child_idx), x=t(b.x), xr=t(b.x_row), g=t(b.gamma))
            for b in batches]
    maxV = max(b.V for b in batches)
    maxX = max(b.n_x for b in batches)
    ctx = Context(b0.cell, b0.N, b0.h, b0.d, precision=args.precision, max_graphs=max(b.K for b in batches),
                  max_vertices=maxV, max_x=maxX, device=local)
    path_info = ctx.path_info()
    h_out = torch.empty(maxV, b0.h, device=dev)
    dparams = torch.empty(ctx.P, device=dev)
    dx = torch.empty(maxX, b0.d, device=dev)
    # N > 1: weight blocks all-reduced on a side stream as soon as the lazy GEMMs finish (overlapping
    # dX and db), the bias block after the backward (dp.BucketedAllReduce)
    allreduce = dp.BucketedAllReduce(ctx, dparams, dp.bias_floats(b0.cell, b0.N, b0.h)) if world > 1 else None

    def step(i):
        p = pool[i % len(pool)]
        V = p["cp"].shape[0] - 1
        ctx.load_graphs(p["gp"], p["cp"], p["ci"])
        ctx.schedule(wait=False)            # header consumed inside forward, overlapping the pull
        if args.inference:
            ctx.forward_inference(params, p["x"], p["xr"], h_out[:V])
            return
        ctx.forward(params, p["x"], p["xr"], h_out[:V])
        ctx.backward(p["g"], dparams, dx[:p["x"].shape[0]])
        if allreduce is not None:
            allreduce.launch()
            allreduce.wait()

    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    ctx.profile(True)
    launches0 = ctx.launches
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for k in range(args.steps):
        if not args.no_flush:
            flush_buf.zero_()                      # L2 flush between timed steps (outside the events)
        ev[k][0].record(stream)
        step(args.warmup + k)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = ctx.launches - launches0
    prof = ctx.profile_read()
    ctx.profile(False)
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    samples = world * b0.K if args.weak else glob[0].K      # graphs the whole job processed per step
    value = samples / (ms / 1000.0)

    # ---- the same steps as CUDA-graph replays (sync-free mode: the host never reads the schedule;
    #      one graph per pool batch captures load + schedule + forward + backward) ----
    graph_line = None
    if world == 1 and not args.inference and not args.no_graph:
        try:
            ctx.set_sync_free(True)
        except Exception as e:                      # path without sync-free support (e.g. h > 512)
            graph_line = {"unavailable": str(e)[:120]}
        if graph_line is None:
            side = torch.cuda.Stream(dev)
            graphs = []
            for i in range(len(pool)):
                g = torch.cuda.CUDAGraph()
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    with torch.cuda.graph(g, stream=side):
                        ctx.set_stream(side)
                        step(i)
                graphs.append(g)
            ctx.set_stream(stream)
            for i in range(args.warmup):
                graphs[i % len(graphs)].replay()
            torch.cuda.synchronize()
            gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for k in range(args.steps):
                if not args.no_flush:
                    flush_buf.zero_()
                gev[k][0].record(stream)
                graphs[(args.warmup + k) % len(graphs)].replay()
                gev[k][1].record(stream)
            torch.cuda.synchronize()
            ctx.sync()                              # the steps' deferred status (valid batches: OK)
            g_ms = sum(a.elapsed_time(b) for a, b in gev) / args.steps
            graph_line = {"value": samples / (g_ms / 1000.0), "unit": "samples/s", "ms_per_step": g_ms,
                          "note": "cavs_set_sync_free + one CUDA graph per pool batch (load, schedule, forward, "
                                  "backward captured); replays timed like the eager steps (CUDA events per step, "
                                  "L2 flushed between steps)"}
            ctx.set_sync_free(False)
            del graphs
    eager_line = {"value": value, "ms_per_step": ms,
                  "note": "the same steps launched eagerly (the host reads each batch's schedule header); the "
                          "phase split and roofline below are measured on this pass"}
    if graph_line and "value" in graph_line:       # headline: the graph replays (same kernels, no host gaps)
        value, ms = graph_line["value"], graph_line["ms_per_step"]

    # ---- roofline of the dominant tensor-core phase (per launch = totals / launches) ----
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    dom = max(TENSOR_PHASES, key=lambda ph: prof[ph]["ms"])
    P = prof[dom]
    achieved = P["flops"] / (P["ms"] / 1000.0) / 1e12 if P["ms"] > 0 else 0.0
    if args.precision == "bf16":
        peak = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops")
        peak_src = "measured (MEASURED_PEAKS.json bf16_tflops_sustained)" if peak else None
        if not peak:
            peak, peak_src = 1400.0, "fallback (B200_PROFILING.md sustained 1.4 PFLOP/s)"
    elif "bf16x3" in path_info:
        # FP32 mode on the tensor cores: every fp32 product is six bf16 tcgen05 MMAs (bf16x3 split
        # operands), so the fp32 roofline is the measured bf16 peak / 6
        bp = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1400.0
        peak = bp / 6.0
        peak_src = ("measured bf16 sustained peak (MEASURED_PEAKS.json) / 6: six bf16 MMAs per fp32 product "
                    "(bf16x3 split)")
    else:
        # FFMA fp32 peak: 148 SMs x 128 FP32 lanes x 2 FLOP x measured max SM clock
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak, peak_src = 148 * 128 * 2 * mhz * 1e6 / 1e12, "derived FFMA peak (148 SM x 128 lanes x 2 x max clock)"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath))
        traffic = tr.get(f"{args.config}:{args.precision}:{dom}")
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic, "peak_source": peak_src,
                "launches": P["launches"], "avg_launch_us": 1000 * P["ms"] / max(1, P["launches"]),
                "pass": "eager steps (library per-phase CUDA events on the launching stream)"}
    phases = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                  "TFLOP/s": (v["flops"] / (v["ms"] / 1000) / 1e12) if v["ms"] > 0 and v["flops"] else None,
                  "GB/s": (v["bytes"] / (v["ms"] / 1000) / 1e9) if v["ms"] > 0 and v["bytes"] else None}
              for k, v in prof.items()}

    # ---- end to end through the C-ABI with HOST buffers ----
    e2e = None
    if not args.no_e2e and not args.inference:
        hb = batches[0]
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hp = dict(gp=pin(hb.graph_ptr), cp=pin(hb.child_ptr), ci=pin(hb.child_idx), pr=pin(params.cpu().numpy()),
                  x=pin(hb.x), xr=pin(hb.x_row), g=pin(hb.gamma))
        # the cotangent rows of the loss vertices (roots for trees, every step for chains): the
        # pipelined entry takes Gamma as rows + values (cavs_train_step_host_async)
        g_rows = np.nonzero(np.abs(hb.gamma).sum(axis=1))[0].astype(np.int32)
        hpa = dict(hp, g=pin(hb.gamma[g_rows]), grow=pin(g_rows))
        hdp = torch.empty(ctx.P, dtype=torch.float32).pin_memory()
        h2d = sum(v.numel() * v.element_size() for v in (hpa if world == 1 else hp).values())
        d2h = hdp.numel() * 4
        dv = {k: torch.empty_like(v, device=dev) for k, v in hp.items()}

        def e2e_sync_step():                        # one synchronous C-ABI call: H2D, step, D2H
            ctx.train_step_host(hp["gp"], hp["cp"], hp["ci"], hp["pr"], hp["x"], hp["xr"], hp["g"], hdp)

        def e2e_step():
            if world == 1:                          # pipelined C-ABI call: H2D of this step overlaps the last
                ctx.train_step_host_async(hpa["gp"], hpa["cp"], hpa["ci"], hpa["pr"], hpa["x"], hpa["xr"], hpa["g"],
                                          hdp, gamma_rows=hpa["grow"])
                return
            for k, v in hp.items():                 # N > 1: the same copies around the data-parallel step
                dv[k].copy_(v, non_blocking=True)
            V = dv["cp"].shape[0] - 1
            ctx.load_graphs(dv["gp"], dv["cp"], dv["ci"])
            ctx.schedule(wait=False)
            ctx.forward(dv["pr"], dv["x"], dv["xr"], h_out[:V])
            ctx.backward(dv["g"], dparams, dx[:dv["x"].shape[0]])
            allreduce.launch()
            allreduce.wait()
            hdp.copy_(dparams, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

        e2e_sync_free = False
        if world == 1:
            try:                                    # the pipelined steps never wait for a schedule header
                ctx.set_sync_free(True)
                e2e_sync_free = True
            except Exception:
                pass
        for _ in range(max(1, args.warmup)):
            e2e_step()
        if world == 1:
            ctx.sync()
        e_steps = max(3, args.steps // 2)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        if world == 1:
            ctx.sync()                              # every step's dparams are on the host
        e_ms = 1000 * (time.perf_counter() - t0) / e_steps
        if e2e_sync_free:
            ctx.set_sync_free(False)
        sync_ms = None
        if world == 1:                              # context: the synchronous single-call step
            e2e_sync_step()
            t0 = time.perf_counter()
            for _ in range(e_steps):
                e2e_sync_step()
            sync_ms = 1000 * (time.perf_counter() - t0) / e_steps
        if world > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": samples / (e_ms / 1000), "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "note": ("cavs_train_step_host_async (two steps in flight: the next step's H2D overlaps this "
                        "step's compute; Gamma as the loss vertices' rows" +
                        ("; sync-free mode" if world == 1 and e2e_sync_free else "") + ")" if world == 1 else
                        "copies + step + bucketed NCCL all-reduce, synchronised each step") +
                       ": pinned host CSR/params/x/x_row/Gamma -> device, schedule, fwd, bwd, "
                       "dparams -> host every step (host wall clock over the steps, max over ranks)"}
        if sync_ms:
            e2e["sync_single_call"] = {"value": samples / (sync_ms / 1000), "ms_per_step": sync_ms,
                                       "h2d_bytes_per_step": int(sum(v.numel() * v.element_size() for v in hp.values())),
                                       "note": "cavs_train_step_host: dense Gamma, synchronised every step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.inference:
        cpu = cpu_baseline(args, b0.K)

    if rank == 0:
        metric = {"tree_lstm": "Tree-LSTM train samples/s (fwd+bwd)", "tree_fc": "Tree-FC train samples/s (fwd+bwd)"}
        line = {
            "metric": (metric[b0.cell] if args.config != "cfg2" and args.config != "cfg3"
                       else "LSTM train samples/s (fwd+bwd)").replace(
                           "train samples/s (fwd+bwd)", "inference samples/s (fwd only)" if args.inference else
                           "train samples/s (fwd+bwd)"),
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": f"{args.config}: {_desc(args.config, b0.h)}", "h": b0.h, "d": b0.d,
                       "batch_per_gpu": float(np.mean([b.K for b in batches])), "global_batch": samples,
                       "precision": args.precision, "engine": path_info,
                       "batch_pool": args.pool, "l2_flush": not args.no_flush, "parallelism": f"dp{world}",
                       "mean_vertices": float(np.mean([b.V for b in batches])),
                       "mean_levels_T": depth_T},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "graph": graph_line,
            "eager": eager_line,
            "clocks": clk,
            "phases": phases,
            "context": "paper (Titan X GM200, CUDA 8, precision not stated, SST): Cavs Tree-LSTM bs=256 "
                       "computation-only 8544/2.3 s = 3,715 samples/s (Table 1, P:L670) — context, not this workload",
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Batched vs serial execution (Fig. 10 / P:L679-694, §8(f) NEXT-1): the same 256-tree
cfg4 batch run as ONE level-batched step (all graphs' tasks merged) and as 256 steps of one graph
each (the serial policy: every task holds a single graph's vertices), device time by CUDA events.

    python tools/serial_vs_batched.py [--config cfg4] [--graphs 256]
    python tools/serial_vs_batched.py --config cfg2 --sweep 2,4,8,16,32,64,128
        Fig. 10's curve: for each batch size bs, one level-batched step over bs graphs vs bs
        single-graph steps (Fixed-LSTM chains of 64, h = 512: the paper's 1.7x ... 36x axis).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1712_04048_b200 import Context
from workloads import gen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--graphs", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sweep", default=None, help="comma-separated batch sizes (graphs per step)")
    ap.add_argument("--precision", default="bf16")
    a = ap.parse_args()
    if a.sweep:
        for bs in [int(x) for x in a.sweep.split(",")]:
            one(a, bs)
        return
    one(a, a.graphs)


def one(a, K_req):
    dev = torch.device("cuda", 0)
    b = gen.make_config_batch(a.config, seed=0, K=K_req if a.config == "cfg2" and K_req > 64 else None)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    K = min(K_req, b.K)
    if K < b.K:                                   # the batched step runs exactly the first K graphs
        gp, cp, ci, rows, recs, nxr = gen.subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, list(range(K)))
        b = gen.Batch(cell=b.cell, N=b.N, h=b.h, d=b.d, graph_ptr=gp, child_ptr=cp, child_idx=ci, x_row=nxr,
                      x=np.ascontiguousarray(b.x[recs]), params=b.params, gamma=np.ascontiguousarray(b.gamma[rows]))
    ctx = Context(b.cell, b.N, b.h, b.d, precision=a.precision, max_graphs=b.K, max_vertices=b.V,
                  max_x=max(1, b.n_x))
    params = t(b.params)
    # per-graph sub-batches (CSR slices re-based to vertex 0, x rows re-indexed)
    subs = []
    for k in range(K):
        lo, hi = int(b.graph_ptr[k]), int(b.graph_ptr[k + 1])
        cp = b.child_ptr[lo:hi + 1] - b.child_ptr[lo]
        ci = b.child_idx[b.child_ptr[lo]:b.child_ptr[hi]]
        xr = b.x_row[lo:hi]
        has = xr >= 0
        x = b.x[xr[has]] if has.any() else np.zeros((0, b.d), np.float32)
        xr2 = np.where(has, np.cumsum(has) - 1, -1).astype(np.int32)
        subs.append(dict(gp=t(np.array([0, hi - lo], np.int32)), cp=t(cp.astype(np.int32)), ci=t(ci.astype(np.int32)),
                         x=t(x.astype(np.float32)) if len(x) else torch.zeros(0, b.d, device=dev), xr=t(xr2),
                         g=t(b.gamma[lo:hi])))
    full = dict(gp=t(b.graph_ptr), cp=t(b.child_ptr), ci=t(b.child_idx), x=t(b.x), xr=t(b.x_row), g=t(b.gamma))

    def run(p):
        ctx.load_graphs(p["gp"], p["cp"], p["ci"])
        ctx.schedule(wait=False)
        ctx.forward(params, p["x"], p["xr"])
        ctx.backward(p["g"])

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    batched = timed(lambda: run(full))
    serial = timed(lambda: [run(s) for s in subs])
    out = {"config": a.config, "precision": a.precision, "graphs": K, "batched_ms": batched, "serial_ms": serial,
           "batched_samples_per_s": b.K / (batched / 1e3), "serial_samples_per_s": K / (serial / 1e3),
           "speedup": serial / batched * (b.K / K)}
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

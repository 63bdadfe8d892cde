"""Shared helpers of the GPU parity tests: run a workloads.Batch through the C-ABI
(via the binding) and through the oracle, and compare (reading Z12: per-tensor
relative 2-norm error ||gpu - ref|| / ||ref||)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from workloads import gen


def rel(a, r):
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    n = np.linalg.norm(r)
    return float(np.linalg.norm(a - r) / (n if n > 0 else 1.0))


def param_blocks(b):
    """Named blocks of the packed parameter vector."""
    h, d, N = b.h, b.d, b.N
    if b.cell == "tree_lstm":
        sizes = [("W", 4 * h * d), ("U_iou", 3 * h * h), ("U_f", h * h), ("b", 4 * h)]
    else:
        sizes = [("W_c", 2 * h * h), ("W_x", h * d), ("b", h)]
    out, o = [], 0
    for n, s in sizes:
        out.append((n, slice(o, o + s)))
        o += s
    return out


def make_ctx(b, precision, max_vertices=None, max_graphs=None, max_x=None):
    from paper_1712_04048_b200 import Context
    return Context(b.cell, b.N, b.h, b.d, precision=precision,
                   max_graphs=max_graphs or b.K, max_vertices=max_vertices or b.V,
                   max_x=max_x if max_x is not None else max(1, b.n_x))


def run_gpu(b, precision="fp32", ctx=None, on_device=True):
    dev = torch.device("cuda", 0)
    if ctx is None:
        ctx = make_ctx(b, precision)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if on_device:
        ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
    else:
        ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    T = ctx.schedule()
    x = t(b.x) if b.n_x else torch.zeros(0, b.d, device=dev)
    h_out = ctx.forward(t(b.params), x, t(b.x_row))
    dparams, dx = ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
    return dict(T=T, h_out=h_out.cpu().numpy(), dparams=dparams.cpu().numpy(),
                dx=dx.cpu().numpy() if dx is not None else None, ctx=ctx)


def run_oracle(b, emulate_bf16=False):
    h_out, dparams, dx, tape = oracle.run(b, emulate_bf16=emulate_bf16)
    return dict(h_out=h_out, dparams=dparams, dx=dx, tape=tape)


def compare(b, g, r, tol, what=""):
    errs = {"h_out": rel(g["h_out"], r["h_out"])}
    for name, sl in param_blocks(b):
        errs["d" + name] = rel(g["dparams"][sl], r["dparams"][sl])
    if b.n_x:
        errs["dx"] = rel(g["dx"], r["dx"])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"{what} errors above {tol}: {bad} (all: {errs})"
    return errs

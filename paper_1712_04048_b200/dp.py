"""Data parallelism across GPUs of one node (torch.distributed over NCCL / NVLink).

The K graphs of a minibatch are independent and F's parameters are
shared, so the batch shards by graph: every rank loads and schedules its own shard with
its own context, and the only exchange step is the all-reduce (sum) of the fp32 weight
gradients (BASELINE.json north_star).  Host-side logic here is covered by the gloo
world_size-2 tests in tests/test_dp_gloo.py.
"""
from __future__ import annotations

import numpy as np

from workloads.gen import subset_csr  # noqa: F401  (re-export: CSR slicing lives with the input generators)


def shard_graphs(sizes, depths, world: int) -> list[list[int]]:
    """Greedy balance of vertex count across ranks (largest graphs first, depth tie-break),
    returning for every rank the ascending list of its graph indices."""
    order = sorted(range(len(sizes)), key=lambda k: (-int(sizes[k]), -int(depths[k]), k))
    load = [0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for k in order:
        r = min(range(world), key=lambda i: (load[i], i))
        parts[r].append(k)
        load[r] += int(sizes[k])
    return [sorted(p) for p in parts]


def graph_depths(graph_ptr, child_ptr, child_idx) -> list[int]:
    """Levels of every graph (1 + the longest child chain): the balance tie-break of shard_graphs.
    Host-side integer work on the CSR (each graph's vertices in a topological pass)."""
    gp = np.asarray(graph_ptr)
    cp = np.asarray(child_ptr)
    ci = np.asarray(child_idx)
    out = []
    for g in range(len(gp) - 1):
        lo, hi = int(gp[g]), int(gp[g + 1])
        n = hi - lo
        ch = [ci[cp[lo + v]:cp[lo + v + 1]].tolist() for v in range(n)]
        lev = [-1] * n
        for v0 in range(n):
            stack = [v0]
            while stack:                              # iterative post-order
                v = stack[-1]
                if lev[v] >= 0:
                    stack.pop()
                    continue
                todo = [c for c in ch[v] if lev[c] < 0]
                if todo:
                    stack.extend(todo)
                else:
                    lev[v] = 1 + max((lev[c] for c in ch[v]), default=-1)
                    stack.pop()
        out.append(1 + max(lev, default=-1))
    return out


def shard_batch(b, world: int, rank: int):
    """This rank's share of ONE global batch `b` (a workloads.Batch): its graphs by shard_graphs,
    re-indexed as a self-contained batch (CSR, pull records, cotangents).  Returns (batch, graphs)."""
    from workloads import gen
    sizes = np.diff(np.asarray(b.graph_ptr))
    parts = shard_graphs(sizes, graph_depths(b.graph_ptr, b.child_ptr, b.child_idx), world)
    mine = parts[rank]
    gp, cp, ci, rows, recs, nxr = subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, mine)
    sb = gen.Batch(cell=b.cell, N=b.N, h=b.h, d=b.d, graph_ptr=gp, child_ptr=cp, child_idx=ci, x_row=nxr,
                   x=np.ascontiguousarray(b.x[recs]), params=b.params, gamma=np.ascontiguousarray(b.gamma[rows]))
    return sb, mine


class BucketedAllReduce:
    """All-reduce (sum) of the packed fp32 dparams in two buckets, overlapped with the backward.

    Bucket 0 = every weight block (all of dparams but the trailing bias block of `n_bias` floats): the
    library records `event` as soon as those are final (cavs_set_grad_event, right after the lazy
    weight-gradient GEMMs), and the bucket is reduced on a side stream while dX and db still run.
    Bucket 1 = the bias block, reduced once the backward is done.  `wait()` makes the caller's
    current stream wait for both.  On CPU tensors (gloo) the buckets are reduced one after the
    other (same result)."""

    def __init__(self, ctx, dparams, n_bias: int, group=None):
        import torch
        self.dparams, self.group = dparams, group
        self.nw = dparams.numel() - n_bias
        self.cuda = dparams.is_cuda
        self.ev = self.side = None
        if self.cuda and ctx is not None:
            self.ev = torch.cuda.Event()
            ctx.set_grad_event(self.ev)
            self.side = torch.cuda.Stream(device=dparams.device)
        self.works = []

    def launch(self):
        """Call right after ctx.backward(...) was enqueued."""
        import torch
        import torch.distributed as dist
        if not (dist.is_initialized() and dist.get_world_size() > 1):
            return
        w, b = self.dparams[:self.nw], self.dparams[self.nw:]
        if self.side is not None:
            with torch.cuda.stream(self.side):
                self.side.wait_event(self.ev)
                self.works.append(dist.all_reduce(w, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(w, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        self.works.append(dist.all_reduce(b, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self):
        for wk in self.works:
            wk.wait()
        self.works = []


def bias_floats(cell: str, N: int, h: int) -> int:
    """Length of the trailing bias block of the packed parameters (include/cavs.h layout)."""
    return 4 * h if cell == "tree_lstm" else h


def allreduce_grads(dparams, group=None):
    """Sum the packed fp32 weight gradients over all ranks (NCCL over NVLink on GPUs,
    gloo in the CPU tests).  In place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(dparams, op=dist.ReduceOp.SUM, group=group)
    return dparams

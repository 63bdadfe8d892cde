"""Data parallelism across GPUs of one node (torch.distributed over NCCL / NVLink).

The K graphs of a minibatch are independent and F's parameters are
shared, so the batch shards by graph: every rank loads and schedules its own shard with
its own context, and the only exchange step is the all-reduce (sum) of the fp32 weight
gradients (BASELINE.json north_star).  Host-side logic here is covered by the gloo
world_size-2 tests in tests/test_dp_gloo.py.
"""
from __future__ import annotations

import numpy as np


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


def subset_csr(graph_ptr, child_ptr, child_idx, x_row, keep):
    """CSR / x_row of the graphs `keep` (in that order); child ids stay instance-local.
    Returns (graph_ptr, child_ptr, child_idx, vertex_rows, x_records) where vertex_rows
    are the kept global vertex ids and x_records the kept pull-record indices."""
    gp = np.asarray(graph_ptr)
    cp = np.asarray(child_ptr)
    rows = np.concatenate([np.arange(gp[k], gp[k + 1]) for k in keep]) if len(keep) else np.zeros(0, np.int64)
    sizes = [int(gp[k + 1] - gp[k]) for k in keep]
    ngp = np.zeros(len(keep) + 1, np.int32)
    ngp[1:] = np.cumsum(sizes)
    deg = (cp[rows + 1] - cp[rows]).astype(np.int32)
    ncp = np.zeros(len(rows) + 1, np.int32)
    ncp[1:] = np.cumsum(deg)
    nci = np.concatenate([child_idx[cp[v]:cp[v + 1]] for v in rows]).astype(np.int32) if len(rows) else \
        np.zeros(0, np.int32)
    xr = np.asarray(x_row)[rows]
    recs = xr[xr >= 0]
    nxr = np.where(xr >= 0, np.cumsum(xr >= 0) - 1, -1).astype(np.int32)
    return ngp, ncp, nci, rows, recs, nxr


def allreduce_grads(dparams, group=None):
    """Sum the packed fp32 weight gradients over all ranks (NCCL over NVLink on GPUs,
    gloo in the CPU tests).  In place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(dparams, op=dist.ReduceOp.SUM, group=group)
    return dparams

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


def allreduce_grads(dparams, group=None):
    """Sum the packed fp32 weight gradients over all ranks (NCCL over NVLink on GPUs,
    gloo in the CPU tests).  In place."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(dparams, op=dist.ReduceOp.SUM, group=group)
    return dparams

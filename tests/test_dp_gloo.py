"""Data-parallel host logic on CPU (gloo, world_size 2): sharding by graph + the gradient
all-reduce reproduce the single-process full-batch gradient.  The fp64 oracle stands in
for the device path on each rank (the GPU path of one rank is covered by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1712_04048_b200 import dp
from workloads import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch():
    return gen.make_batch("tree_lstm", 2, 6, 5, "sst_tree", 9, seed=21)


def _rank_grad(b, keep):
    gp, cp, ci, rows, recs, nxr = dp.subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, keep)
    sb = gen.Batch(cell=b.cell, N=b.N, h=b.h, d=b.d, graph_ptr=gp, child_ptr=cp, child_idx=ci, x_row=nxr,
                   x=b.x[recs], params=b.params, gamma=b.gamma[rows])
    _, dparams, _, _ = oracle.run(sb)
    return dparams


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = _batch()
    sizes = np.diff(b.graph_ptr)
    parts = dp.shard_graphs(sizes, sizes, world)
    g = torch.from_numpy(_rank_grad(b, parts[rank]))
    dp.allreduce_grads(g)
    out[rank] = g.numpy().copy()
    dist.destroy_process_group()


def test_shard_graphs_partition_and_balance():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 111, size=256)
    for world in (1, 2, 4, 8):
        parts = dp.shard_graphs(sizes, sizes, world)
        flat = sorted(k for p in parts for k in p)
        assert flat == list(range(256))
        loads = [int(sizes[p].sum()) for p in parts]
        assert max(loads) - min(loads) <= sizes.max()


def test_subset_csr_roundtrip():
    b = _batch()
    keep = [1, 4, 7]
    gp, cp, ci, rows, recs, nxr = dp.subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, keep)
    assert gp[-1] == len(rows) == cp.size - 1
    assert ci.size == cp[-1]
    assert np.array_equal(b.x[recs], b.x[b.x_row[rows][b.x_row[rows] >= 0]])


@pytest.mark.timeout(300)
def test_gloo_allreduce_equals_full_batch_gradient():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    _, full, _, _ = oracle.run(_batch())
    for r in range(world):
        np.testing.assert_allclose(out[r], full, rtol=1e-10, atol=1e-12)


def test_graph_depths_match_the_oracle_levels():
    b = _batch()
    lv = oracle.levels_recursive(oracle.global_children(b.graph_ptr, b.child_ptr, b.child_idx))
    want = [int(lv[b.graph_ptr[k]:b.graph_ptr[k + 1]].max()) + 1 for k in range(b.K)]
    assert dp.graph_depths(b.graph_ptr, b.child_ptr, b.child_idx) == want


def test_shard_batch_covers_the_global_batch():
    """Strong scaling: the shards of ONE global batch are disjoint, cover every graph,
    and each is a self-contained batch whose oracle outputs equal the full batch's rows."""
    b = _batch()
    ho, _, _, _ = oracle.run(b, with_backward=False)
    seen = []
    for world in (3, 4):
        seen = []
        for r in range(world):
            sb, mine = dp.shard_batch(b, world, r)
            seen += mine
            hs, _, _, _ = oracle.run(sb, with_backward=False)
            rows = np.concatenate([np.arange(b.graph_ptr[k], b.graph_ptr[k + 1]) for k in mine])
            np.testing.assert_array_equal(hs, ho[rows])
        assert sorted(seen) == list(range(b.K))


def _worker_bucketed(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = _batch()
    sb, _ = dp.shard_batch(b, world, rank)
    _, dparams, _, _ = oracle.run(sb)
    g = torch.from_numpy(dparams)
    ar = dp.BucketedAllReduce(None, g, dp.bias_floats(b.cell, b.N, b.h))
    ar.launch()
    ar.wait()
    out[rank] = g.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_bucketed_allreduce_4_uneven_ranks():
    """world_size 4 over 9 graphs (uneven shards): the two-bucket all-reduce of the sharded
    gradients equals the single-process full-batch gradient (graphs independent)."""
    world = 4
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_bucketed, args=(world, _free_port(), out), nprocs=world, join=True)
    _, full, _, _ = oracle.run(_batch())
    for r in range(world):
        np.testing.assert_allclose(out[r], full, rtol=1e-10, atol=1e-12)

"""Generator unit tests: determinism, sizes, CSR well-formedness."""
import numpy as np

from workloads import gen


def test_determinism():
    a = gen.make_config_batch("cfg4", seed=3, K=16, h=8)
    b = gen.make_config_batch("cfg4", seed=3, K=16, h=8)
    for f in ("graph_ptr", "child_ptr", "child_idx", "x_row", "x", "params", "gamma"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_remy_sizes_and_shape():
    rng = np.random.default_rng(0)
    for L in (1, 2, 3, 8, 56):
        ch = gen.remy_tree(L, rng)
        assert len(ch) == 2 * L - 1
        assert sum(1 for c in ch if not c) == L
        assert all(len(c) in (0, 2) for c in ch)
        parents = [p for c in ch for p in c]
        assert len(set(parents)) == len(parents) == 2 * L - 2


def test_cbt_and_chain():
    ch = gen.complete_binary_tree(256)
    assert len(ch) == 511
    assert gen.chain(3) == [[], [0], [1]]


def test_csr_wellformed_and_x_policy():
    b = gen.make_config_batch("cfg4", seed=0, K=32, h=8)
    assert b.graph_ptr[0] == 0 and np.all(np.diff(b.graph_ptr) >= 1)
    assert b.child_ptr[0] == 0 and np.all(np.diff(b.child_ptr) >= 0)
    assert b.child_ptr[-1] == b.child_idx.size == b.V - b.K
    deg = np.diff(b.child_ptr)
    assert np.array_equal(b.x_row >= 0, deg == 0)          # x at leaves
    is_child = np.zeros(b.V, bool)                          # the loss is at the roots (Z9)
    for g in range(b.K):
        lo, hi = b.graph_ptr[g], b.graph_ptr[g + 1]
        for v in range(lo, hi):
            is_child[lo + b.child_idx[b.child_ptr[v]:b.child_ptr[v + 1]]] = True
    assert b.gamma[~is_child].any(axis=1).all() and not b.gamma[is_child].any()
    c = gen.make_config_batch("cfg3", seed=0, K=8, h=8)
    assert np.all(c.x_row >= 0)                               # chains: x everywhere
    lens = gen.sst_lengths(10000, np.random.default_rng(1))
    assert lens.min() >= 1 and lens.max() <= 56 and 17 < lens.mean() < 21

"""Seeded graph / input / parameter generators (no method arithmetic here).

Recipe:
  * graph shapes from seed s, params from s+1 ~ U(-0.1, 0.1),
    inputs x from s+2 ~ U(-1, 1), cotangents Gamma from s+3 ~ N(0, 1);
  * local vertex ids are a random permutation per graph, so nothing may rely
    on topologically ordered ids;
  * trees carry x at their leaves (word inputs), chains at every vertex;
  * loss vertices (nonzero Gamma) are the roots of trees and every vertex of
    chains (PAPER.md P:L606 next-word LM, P:L609 sentiment at the root).

Shapes follow the paper's workloads: complete binary trees with 256 leaves
(P:L608, 511 vertices), chains of 64 steps, SST-shaped binarised
parse trees / sentences with lengths ~ round(Gamma(mean 19, sd 9)) clipped to
[1, 56] (BASELINE.json configs; SST's longest sentence is 54-56 words,
P:L609 / P:L638), tree shapes drawn Remy-uniform over full binary trees.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CELL_TREE_LSTM = "tree_lstm"
CELL_TREE_FC = "tree_fc"


def n_params(cell: str, N: int, h: int, d: int) -> int:
    """Length of the packed fp32 parameter vector (layout in include/cavs.h)."""
    if cell == CELL_TREE_LSTM:
        return 4 * h * d + 3 * h * h + h * h + 4 * h
    if cell == CELL_TREE_FC:
        return h * 2 * h + h * d + h
    raise ValueError(cell)


# --------------------------------------------------------------------------
# graph shapes: each returns a list of child lists over local ids 0..n-1
# --------------------------------------------------------------------------
def remy_tree(n_leaves: int, rng: np.random.Generator) -> list[list[int]]:
    """Uniformly random full binary tree with `n_leaves` leaves (Remy's algorithm)."""
    if n_leaves < 1:
        raise ValueError("n_leaves >= 1")
    parent = [-1]
    children: list[list[int]] = [[]]
    for _ in range(n_leaves - 1):
        x = int(rng.integers(len(children)))
        n = len(children)          # new internal vertex
        leaf = n + 1               # new leaf
        children.append([])
        children.append([])
        parent.extend([-1, -1])
        p = parent[x]
        if p >= 0:
            children[p][children[p].index(x)] = n
        parent[n] = p
        if rng.integers(2) == 0:
            children[n] = [x, leaf]
        else:
            children[n] = [leaf, x]
        parent[x] = n
        parent[leaf] = n
    return children


def complete_binary_tree(n_leaves: int) -> list[list[int]]:
    """Complete binary tree: leaves 0..L-1, internal vertices appended level by level,
    root last."""
    if n_leaves < 1 or (n_leaves & (n_leaves - 1)):
        raise ValueError("n_leaves must be a power of two")
    children: list[list[int]] = [[] for _ in range(n_leaves)]
    prev = list(range(n_leaves))
    while len(prev) > 1:
        cur = []
        for i in range(0, len(prev), 2):
            children.append([prev[i], prev[i + 1]])
            cur.append(len(children) - 1)
        prev = cur
    return children


def chain(n: int) -> list[list[int]]:
    """Chain 0 -> 1 -> ... -> n-1: children(i) = [i-1]."""
    if n < 1:
        raise ValueError("n >= 1")
    return [[]] + [[i - 1] for i in range(1, n)]


def permute(children: list[list[int]], rng: np.random.Generator) -> list[list[int]]:
    """Relabel vertices with a random permutation (child order within a list kept)."""
    n = len(children)
    perm = rng.permutation(n)            # old id -> new id
    out: list[list[int]] = [[] for _ in range(n)]
    for old, ch in enumerate(children):
        out[int(perm[old])] = [int(perm[c]) for c in ch]
    return out


def sst_lengths(k: int, rng: np.random.Generator, lo: int = 1, hi: int = 56) -> np.ndarray:
    """Sentence lengths ~ round(Gamma(mean 19, sd 9)) clipped to [lo, hi]."""
    mean, sd = 19.0, 9.0
    shape = (mean / sd) ** 2
    scale = sd * sd / mean
    return np.clip(np.rint(rng.gamma(shape, scale, size=k)), lo, hi).astype(np.int64)


# --------------------------------------------------------------------------
# batches
# --------------------------------------------------------------------------
@dataclass
class Batch:
    cell: str
    N: int
    h: int
    d: int
    graph_ptr: np.ndarray          # int32 [K+1] global vertex offsets
    child_ptr: np.ndarray          # int32 [V+1]
    child_idx: np.ndarray          # int32 [E] instance-LOCAL child ids
    x_row: np.ndarray              # int32 [V] record index or -1
    x: np.ndarray                  # float32 [n_x, d]
    params: np.ndarray             # float32 [P]
    gamma: np.ndarray              # float32 [V, h] = dL/dh_push (cotangents)
    is_chain: bool = False
    meta: dict = field(default_factory=dict)

    @property
    def K(self) -> int:
        return int(self.graph_ptr.size - 1)

    @property
    def V(self) -> int:
        return int(self.child_ptr.size - 1)

    @property
    def n_x(self) -> int:
        return int(self.x.shape[0])


def batch_from_graphs(graphs: list[list[list[int]]], *, cell: str, N: int, h: int, d: int,
                      seed: int, x_at: str = "leaves", loss_at: str = "roots",
                      x_values: np.ndarray | None = None, params: np.ndarray | None = None,
                      gamma_scale: float = 1.0) -> Batch:
    """Concatenate per-instance child lists into the CSR the C-ABI takes and draw
    x / params / Gamma from the seed layout.  `x_at` in {"leaves", "all", "none"}."""
    sizes = [len(g) for g in graphs]
    graph_ptr = np.zeros(len(graphs) + 1, dtype=np.int32)
    graph_ptr[1:] = np.cumsum(sizes)
    V = int(graph_ptr[-1])
    child_ptr = np.zeros(V + 1, dtype=np.int32)
    idx: list[int] = []
    has_parent = np.zeros(V, dtype=bool)
    is_leaf = np.zeros(V, dtype=bool)
    v = 0
    for k, g in enumerate(graphs):
        base = int(graph_ptr[k])
        for ch in g:
            idx.extend(ch)
            child_ptr[v + 1] = child_ptr[v] + len(ch)
            is_leaf[v] = len(ch) == 0
            for c in ch:
                if 0 <= c < len(g):      # tolerate invalid ids (validation tests)
                    has_parent[base + c] = True
            v += 1
    child_idx = np.asarray(idx, dtype=np.int32)

    if x_at == "leaves":
        x_mask = is_leaf
    elif x_at == "all":
        x_mask = np.ones(V, dtype=bool)
    elif x_at == "none":
        x_mask = np.zeros(V, dtype=bool)
    else:
        raise ValueError(x_at)
    x_row = np.full(V, -1, dtype=np.int32)
    n_x = int(x_mask.sum())
    x_row[x_mask] = np.arange(n_x, dtype=np.int32)
    if x_values is None:
        rng_x = np.random.default_rng(seed + 2)
        x = rng_x.uniform(-1.0, 1.0, size=(n_x, d)).astype(np.float32)
    else:
        x = np.ascontiguousarray(x_values[:n_x], dtype=np.float32)

    if params is None:
        rng_p = np.random.default_rng(seed + 1)
        params = rng_p.uniform(-0.1, 0.1, size=n_params(cell, N, h, d)).astype(np.float32)

    if loss_at == "roots":
        loss_mask = ~has_parent
    elif loss_at == "all":
        loss_mask = np.ones(V, dtype=bool)
    else:
        raise ValueError(loss_at)
    rng_g = np.random.default_rng(seed + 3)
    gamma = (rng_g.standard_normal(size=(V, h)) * gamma_scale).astype(np.float32)
    gamma[~loss_mask] = 0.0
    return Batch(cell=cell, N=N, h=h, d=d, graph_ptr=graph_ptr, child_ptr=child_ptr,
                 child_idx=child_idx, x_row=x_row, x=x, params=params, gamma=gamma,
                 is_chain=(x_at == "all"))


# BASELINE.json configs.  `K` = graphs per batch.
CONFIGS = {
    "cfg1": dict(cell=CELL_TREE_FC, N=2, h=16, d=16, K=4, shape="remy8",
                 desc="Tree-FC, 4 random binary trees of 8 leaves, hidden 16, fp32"),
    "cfg2": dict(cell=CELL_TREE_LSTM, N=1, h=512, d=512, K=64, shape="chain64",
                 desc="Fixed-LSTM LM, PTB-shaped synthetic tokens, seq len 64, hidden 512, batch 64"),
    "cfg3": dict(cell=CELL_TREE_LSTM, N=1, h=512, d=512, K=256, shape="sst_chain",
                 desc="Var-LSTM, SST-shaped lengths 1-56, hidden 512, batch 256"),
    "cfg4": dict(cell=CELL_TREE_LSTM, N=2, h=512, d=512, K=256, shape="sst_tree",
                 desc="Tree-LSTM, synthetic SST-shaped binarised parse trees, hidden 512, batch 256"),
    "cfg4_h1024": dict(cell=CELL_TREE_LSTM, N=2, h=1024, d=1024, K=256, shape="sst_tree",
                       desc="Tree-LSTM, synthetic SST-shaped binarised parse trees, hidden 1024, batch 256"),
    "cfg5": dict(cell=CELL_TREE_FC, N=2, h=2048, d=2048, K=64, shape="cbt256",
                 desc="Tree-FC, complete binary trees of 256 leaves, hidden 2048, batch 64"),
}


def make_graphs(shape: str, K: int, seed: int) -> list[list[list[int]]]:
    rng = np.random.default_rng(seed)
    if shape.startswith("remy"):
        L = int(shape[4:])
        return [permute(remy_tree(L, rng), rng) for _ in range(K)]
    if shape.startswith("cbt"):
        L = int(shape[3:])
        return [permute(complete_binary_tree(L), rng) for _ in range(K)]
    if shape.startswith("chain"):
        n = int(shape[5:])
        return [permute(chain(n), rng) for _ in range(K)]
    if shape == "sst_tree":
        lens = sst_lengths(K, rng)
        return [permute(remy_tree(int(L), rng), rng) for L in lens]
    if shape == "sst_chain":
        lens = sst_lengths(K, rng)
        return [permute(chain(int(L)), rng) for L in lens]
    raise ValueError(shape)


def _embedding_x(n_x: int, d: int, seed: int, vocab: int = 10000) -> np.ndarray:
    """x = rows of an embedding table U(-0.1,0.1) for Zipf tokens p(r) ~ 1/r over a
    PTB-sized vocabulary ("over 10K different words")."""
    rng = np.random.default_rng(seed + 2)
    table = rng.uniform(-0.1, 0.1, size=(vocab, d)).astype(np.float32)
    p = 1.0 / np.arange(1, vocab + 1)
    p /= p.sum()
    tok = rng.choice(vocab, size=n_x, p=p)
    return table[tok]


@dataclass
class LMBatch:
    """Language-model batch: `batch` is the F-over-G part (chains, N = 1) whose
    pull records are the rows of an embedding table (x = table [vocab, d], x_row[v] = token of
    vertex v: the embedding pull); `targets[v]` = next token of the sequence (-1 at the last step);
    W_out [vocab, h], b_out [vocab]: the softmax head's parameters."""
    batch: "Batch"
    tokens: np.ndarray
    targets: np.ndarray
    W_out: np.ndarray
    b_out: np.ndarray


def make_lm_batch(K: int, lengths, h: int, d: int, vocab: int, seed: int) -> LMBatch:
    """K sequences (lengths: an int or one per sequence) of Zipf tokens p(r) ~ 1/r over `vocab`
    (PTB-sized at 10k), chains 0 -> 1 -> ... (vertex t reads token t, predicts token t+1);
    params U(-0.1, 0.1), embedding and head U(-0.1, 0.1)."""
    rng = np.random.default_rng(seed)
    lens = [int(lengths)] * K if np.isscalar(lengths) else [int(x) for x in lengths]
    p = 1.0 / np.arange(1, vocab + 1)
    p /= p.sum()
    seqs = [rng.choice(vocab, size=n + 1, p=p).astype(np.int32) for n in lens]
    b = batch_from_graphs([chain(n) for n in lens], cell="tree_lstm", N=1, h=h, d=d, seed=seed, x_at="none",
                          loss_at="all")
    b.x = rng.uniform(-0.1, 0.1, size=(vocab, d)).astype(np.float32)
    b.x_row = np.concatenate([q[:-1] for q in seqs]).astype(np.int32)
    targets = np.concatenate([np.concatenate([q[1:-1], [-1]]) for q in seqs]).astype(np.int32)
    W_out = rng.uniform(-0.1, 0.1, size=(vocab, h)).astype(np.float32)
    b_out = rng.uniform(-0.1, 0.1, size=vocab).astype(np.float32)
    return LMBatch(batch=b, tokens=b.x_row.copy(), targets=targets, W_out=W_out, b_out=b_out)


def make_batch(cell: str, N: int, h: int, d: int, shape: str, K: int, seed: int,
               gamma_scale: float = 1.0) -> Batch:
    graphs = make_graphs(shape, K, seed)
    is_chain = shape.startswith("chain") or shape == "sst_chain"
    x_values = None
    if shape.startswith("chain"):
        n_x = sum(len(g) for g in graphs)
        x_values = _embedding_x(n_x, d, seed)
    b = batch_from_graphs(graphs, cell=cell, N=N, h=h, d=d, seed=seed,
                          x_at="all" if is_chain else "leaves",
                          loss_at="all" if is_chain else "roots",
                          x_values=x_values, gamma_scale=gamma_scale)
    b.meta = dict(shape=shape, seed=seed)
    return b


def make_config_batch(name: str, seed: int = 0, K: int | None = None, h: int | None = None,
                      d: int | None = None) -> Batch:
    c = CONFIGS[name]
    hh = h if h is not None else c["h"]
    dd = d if d is not None else (hh if h is not None else c["d"])
    b = make_batch(c["cell"], c["N"], hh, dd, c["shape"], K if K is not None else c["K"], seed)
    b.meta["config"] = name
    return b


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

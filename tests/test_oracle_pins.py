"""Pins for the CPU oracle: what the paper and the mathematics fix.

None of these re-types the oracle's formulas: they compare against closed forms,
brute force (the literal Alg. 1 loop), a library routine (torch.nn.LSTM, torch's
bf16 conversion), finite differences, and hand-worked values (tests/golden/).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.cavs_oracle import global_children
from workloads import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _csr(graphs):
    return gen.batch_from_graphs(graphs, cell="tree_lstm", N=2, h=1, d=1, seed=0)


# ---------------------------------------------------------------- P9 rounding
def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    a = np.concatenate([rng.standard_normal(100000) * 10 ** rng.uniform(-8, 8, 100000),
                        # exact ties at the bf16 rounding boundary
                        (np.arange(1, 2000, dtype=np.float32).view(np.uint32) | 0x8000).view(np.float32)])
    a = a.astype(np.float32)
    ref = torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(oracle.bf16r(a), ref)


# ---------------------------------------------------------------- P1 schedule
def _sizes(level_ptr):
    return list(np.diff(level_ptr))


@pytest.mark.parametrize("shape,K", [("remy8", 4), ("sst_tree", 32), ("sst_chain", 16),
                                     ("cbt16", 3), ("chain7", 5)])
def test_alg1_literal_equals_level_formula(shape, K):
    g = gen.make_graphs(shape, K, seed=3)
    b = _csr(g)
    ch = global_children(b.graph_ptr, b.child_ptr, b.child_idx)
    S = oracle.schedule_alg1(ch)
    level, level_ptr, order = oracle.schedule(ch)
    assert len(S) == len(level_ptr) - 1
    for t, Vt in enumerate(S):
        assert Vt == sorted(Vt)
        assert list(order[level_ptr[t]:level_ptr[t + 1]]) == Vt
        assert all(level[v] == t for v in Vt)


def test_schedule_closed_forms():
    # K complete binary trees with L leaves -> log2(L)+1 tasks of sizes K*L/2^t
    for L, K in [(4, 3), (256, 2), (1, 5)]:
        b = _csr([gen.permute(gen.complete_binary_tree(L), np.random.default_rng(L)) for _ in range(K)])
        _, lp, _ = oracle.schedule(global_children(b.graph_ptr, b.child_ptr, b.child_idx))
        T = int(np.log2(L)) + 1
        assert _sizes(lp) == [K * L // 2 ** t for t in range(T)]
    # 64-step chain x K -> 64 tasks of size K
    b = _csr([gen.permute(gen.chain(64), np.random.default_rng(k)) for k in range(6)])
    _, lp, _ = oracle.schedule(global_children(b.graph_ptr, b.child_ptr, b.child_idx))
    assert _sizes(lp) == [6] * 64
    # var-length {3, 5} -> sizes [2,2,2,1,1]
    b = _csr([gen.chain(3), gen.chain(5)])
    _, lp, _ = oracle.schedule(global_children(b.graph_ptr, b.child_ptr, b.child_idx))
    assert _sizes(lp) == [2, 2, 2, 1, 1]
    # mixed batch of S:L341: chain 0->1->2 and tree {0,1}->2: [{c0,t0,t1},{c1,t2},{c2}]
    b = _csr([gen.chain(3), [[], [], [0, 1]]])
    S = oracle.schedule_alg1(global_children(b.graph_ptr, b.child_ptr, b.child_idx))
    assert S == [[0, 3, 4], [1, 5], [2]]


def test_validation_errors():
    def err(graphs, N=2):
        b = _csr(graphs)
        with pytest.raises(oracle.OracleError) as e:
            oracle.validate(b.graph_ptr, b.child_ptr, b.child_idx, N)
        return e.value.code

    assert err([[[1], [0]]]) == "cycle"
    assert err([[[0]]]) == "cycle"
    assert err([[[1, 2, 3], [], [], []]]) == "arity"
    assert err([[[5], []]]) == "invalid"
    b = _csr([[[]]])
    with pytest.raises(oracle.OracleError):
        oracle.validate(np.array([0, 1, 1], np.int32), b.child_ptr, b.child_idx, 2)
    with pytest.raises(oracle.OracleError) as e:
        b = _csr([[[1, 1], []]])
        oracle.validate(b.graph_ptr, b.child_ptr, b.child_idx, 2, allow_fanout=False)
    assert e.value.code == "fanout"


# ---------------------------------------------------------------- P2 evaluation log
def test_each_vertex_once_after_children():
    b = gen.make_batch("tree_lstm", 2, 4, 3, "sst_tree", 8, seed=1)
    _, tape = oracle.forward(b.cell, b.N, b.h, b.d, b.params, b.graph_ptr, b.child_ptr,
                             b.child_idx, b.x_row, b.x)
    log = tape.log
    assert sorted(log) == list(range(b.V))
    where = {v: i for i, v in enumerate(log)}
    for v, ch in enumerate(tape.children):
        for c in ch:
            assert where[c] < where[v]


# ---------------------------------------------------------------- P3 chain == LSTM
def _lstm_torch_params(P, h, d):
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    lstm = torch.nn.LSTM(d, h, batch_first=False).double()
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(t(np.concatenate([P["W_i"], P["W_f"], P["W_u"], P["W_o"]])))
        lstm.weight_hh_l0.copy_(t(np.concatenate([P["U_i"], P["U_f"], P["U_u"], P["U_o"]])))
        lstm.bias_ih_l0.copy_(t(np.concatenate([P["b_i"], P["b_f"], P["b_u"], P["b_o"]])))
        lstm.bias_hh_l0.zero_()
    return lstm


def test_chain_tree_lstm_equals_torch_lstm():
    h, d = 5, 3
    b = gen.make_batch("tree_lstm", 1, h, d, "sst_chain", 6, seed=7)
    h_out, dparams, dx, tape = oracle.run(b)
    P = oracle.unpack("tree_lstm", 1, h, d, b.params)
    lstm = _lstm_torch_params(P, h, d)
    ch = tape.children
    parent = {c: v for v, cs in enumerate(ch) for c in cs}
    total = 0.0
    for k in range(b.K):
        lo, hi = int(b.graph_ptr[k]), int(b.graph_ptr[k + 1])
        v = next(u for u in range(lo, hi) if not ch[u])       # first step has no child
        seq = [v]
        while seq[-1] in parent:
            seq.append(parent[seq[-1]])
        X = torch.tensor(b.x[b.x_row[seq]], dtype=torch.float64).unsqueeze(1)
        out, _ = lstm(X)
        ref = out[:, 0, :].detach().numpy()
        np.testing.assert_allclose(h_out[seq], ref, rtol=0, atol=1e-14)
        total = total + (out[:, 0, :] * torch.tensor(b.gamma[seq], dtype=torch.float64)).sum()
    total.backward()
    g = {"W": lstm.weight_ih_l0.grad.numpy(), "U": lstm.weight_hh_l0.grad.numpy(),
         "b": lstm.bias_ih_l0.grad.numpy()}
    G = oracle.unpack("tree_lstm", 1, h, d, dparams)
    sl = {"i": slice(0, h), "f": slice(h, 2 * h), "u": slice(2 * h, 3 * h), "o": slice(3 * h, 4 * h)}
    for gate, s in sl.items():
        np.testing.assert_allclose(G["W_" + gate], g["W"][s], atol=1e-12)
        np.testing.assert_allclose(G["U_" + gate], g["U"][s], atol=1e-12)
        np.testing.assert_allclose(G["b_" + gate], g["b"][s], atol=1e-12)


# ---------------------------------------------------------------- P4 special cases
def test_zero_params_give_zero_h():
    b = gen.make_batch("tree_lstm", 2, 4, 4, "sst_tree", 5, seed=2)
    b.params[:] = 0
    b.x[:] = 0
    h_out, _, _, _ = oracle.run(b, with_backward=False)
    assert np.all(h_out == 0)
    bf = gen.make_batch("tree_fc", 2, 4, 4, "remy8", 3, seed=2)
    bf.params[:] = 0
    h_out, _, _, _ = oracle.run(bf, with_backward=False)
    assert np.all(h_out == 0)


def test_leaf_is_lstm_cell_from_zero_state():
    h, d = 6, 4
    b = gen.make_batch("tree_lstm", 2, h, d, "sst_tree", 4, seed=5)
    h_out, _, _, tape = oracle.run(b, with_backward=False)
    P = oracle.unpack("tree_lstm", 2, h, d, b.params)
    cell = torch.nn.LSTMCell(d, h).double()
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(t(np.concatenate([P["W_i"], P["W_f"], P["W_u"], P["W_o"]])))
        cell.weight_hh.zero_()
        cell.bias_ih.copy_(t(np.concatenate([P["b_i"], P["b_f"], P["b_u"], P["b_o"]])))
        cell.bias_hh.zero_()
    leaves = [v for v, c in enumerate(tape.children) if not c]
    X = t(b.x[b.x_row[leaves]])
    hh, cc = cell(X)
    np.testing.assert_allclose(h_out[leaves], hh.detach().numpy(), atol=1e-14)


# ---------------------------------------------------------------- P5 golden examples
def _golden_batch(g):
    gp = np.array([0, len(g["children"])], np.int32)
    b = gen.batch_from_graphs([g["children"]], cell=g["cell"], N=g["N"], h=1, d=1, seed=0, x_at="all")
    b.x = np.array(g["x"], dtype=np.float32).reshape(-1, 1)
    if g["cell"] == "tree_lstm":
        P = {}
        for gate in "ifou":
            P["W_" + gate] = np.array([[g["W"][gate]]])
            P["U_" + gate] = np.array([[g["U"][gate]]])
            P["b_" + gate] = np.array([g["b"][gate]])
        theta = oracle.pack("tree_lstm", 2, 1, 1, P)
    else:
        theta = np.array([g["W_l"], g["W_r"], g["W_x"], g["b"]])
    assert np.array_equal(b.graph_ptr, gp)
    return b, theta


@pytest.mark.parametrize("name", ["w1_tree_lstm", "w2_tree_lstm", "w3_tree_fc"])
def test_golden_three_node(name):
    g = json.load(open(os.path.join(GOLD, name + ".json")))
    b, theta = _golden_batch(g)
    X = np.array(g["x"], dtype=np.float64).reshape(-1, 1)   # fp64 inputs (0.1 etc. exactly as printed)
    h_out, tape = oracle.forward(g["cell"], 2, 1, 1, theta, b.graph_ptr, b.child_ptr, b.child_idx,
                                 b.x_row, X)
    np.testing.assert_allclose(h_out[:, 0], g["expect_h"], rtol=0, atol=g["tol"])
    if "expect_c" in g:
        np.testing.assert_allclose([tape.st[v]["c"][0] for v in range(3)], g["expect_c"], atol=g["tol"])
    if "expect_grad" in g:
        gamma = np.zeros((3, 1))
        gamma[g["loss_vertex"]] = 1.0
        dp, dx = oracle.backward(g["cell"], 2, 1, 1, theta, tape, b.x_row, 3, gamma)
        G = oracle.unpack("tree_lstm", 2, 1, 1, dp)
        eg = g["expect_grad"]
        for gate in "ifou":
            assert abs(G["W_" + gate][0, 0] - eg["W"][gate]) < g["grad_tol"]
            assert abs(G["U_" + gate][0, 0] - eg["U"][gate]) < g["grad_tol"]
            assert abs(G["b_" + gate][0] - eg["b"][gate]) < g["grad_tol"]
        np.testing.assert_allclose(dx[:, 0], eg["x"], atol=g["grad_tol"])


def test_golden_cbt256_symmetry():
    g = json.load(open(os.path.join(GOLD, "w4_tree_fc_cbt256.json")))
    rng = np.random.default_rng(0)
    b = gen.batch_from_graphs([gen.permute(gen.complete_binary_tree(g["leaves"]), rng)],
                              cell="tree_fc", N=2, h=1, d=1, seed=0, x_at="leaves")
    X = np.full((b.n_x, 1), g["leaf_x"])
    theta = np.array([g["W_l"], g["W_r"], g["W_x"], g["b"]])
    h_out, tape = oracle.forward("tree_fc", 2, 1, 1, theta, b.graph_ptr, b.child_ptr, b.child_idx,
                                 b.x_row, X)
    level, lp, order = oracle.schedule(tape.children)
    for t in range(len(lp) - 1):
        vals = h_out[order[lp[t]:lp[t + 1]], 0]
        assert np.all(vals == vals[0])                      # P8: symmetry
        if str(t) in g["expect_level"]:
            assert abs(vals[0] - g["expect_level"][str(t)]) < g["tol"]


# ---------------------------------------------------------------- P6 finite differences
def _fd_case(cell, N, h, d, graphs, seed):
    b = gen.batch_from_graphs(graphs, cell=cell, N=N, h=h, d=d, seed=seed, x_at="all", loss_at="all")
    X = b.x.astype(np.float64)
    theta = b.params.astype(np.float64)
    gamma = b.gamma.astype(np.float64)

    def L(th, Xv):
        ho, _ = oracle.forward(cell, N, h, d, th, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, Xv)
        return oracle.loss(ho, gamma)

    _, tape = oracle.forward(cell, N, h, d, theta, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, X)
    dp, dx = oracle.backward(cell, N, h, d, theta, tape, b.x_row, b.n_x, gamma)
    eps = 1e-6
    num = np.zeros_like(theta)
    for j in range(theta.size):
        e = np.zeros_like(theta); e[j] = eps
        num[j] = (L(theta + e, X) - L(theta - e, X)) / (2 * eps)
    numx = np.zeros_like(X)
    for j in np.ndindex(X.shape):
        e = np.zeros_like(X); e[j] = eps
        numx[j] = (L(theta, X + e) - L(theta, X - e)) / (2 * eps)
    scale = max(1.0, np.abs(num).max())
    assert np.abs(dp - num).max() / scale < 1e-7, np.abs(dp - num).max()
    assert np.abs(dx - numx).max() / max(1.0, np.abs(numx).max()) < 1e-7


@pytest.mark.parametrize("case", ["lstm2", "lstm1_chain", "lstm3", "fc"])
def test_finite_differences(case):
    # 6-vertex tree with a unary vertex (missing child slot), params scaled up so gates saturate less
    tree = [[], [], [0, 1], [], [3], [2, 4]]
    if case == "lstm2":
        _fd_case("tree_lstm", 2, 3, 2, [tree, [[]]], seed=11)
    elif case == "lstm1_chain":
        _fd_case("tree_lstm", 1, 3, 2, [gen.chain(4), gen.chain(2)], seed=12)
    elif case == "lstm3":
        _fd_case("tree_lstm", 3, 2, 2, [[[], [], [], [0, 1, 2], [3]]], seed=13)
    else:
        _fd_case("tree_fc", 2, 3, 2, [tree, [[], [0]]], seed=14)


@pytest.mark.parametrize("case", ["lstm2_dag", "lstm3_dup", "fc_dag"])
def test_finite_differences_dag(case):
    """DAG inputs (NEXT-3; P:L189-191 graph-structured RNNs, P:L447 gradients ADDED): a child shared
    by two parents and a child listed twice by one parent; the oracle's additive backward must equal
    central differences of its own forward (which evaluates a shared child once)."""
    # 0, 1 leaves; 2 = (0, 1); 3 = (1, 2): vertex 1 has two parents; 4 = (3, 3): duplicate child
    dag = [[], [], [0, 1], [1, 2], [3, 3]]
    if case == "lstm2_dag":
        _fd_case("tree_lstm", 2, 3, 2, [dag, [[]]], seed=15)
    elif case == "lstm3_dup":
        _fd_case("tree_lstm", 3, 2, 2, [[[], [], [0, 0, 1], [2, 0]]], seed=16)
    else:
        _fd_case("tree_fc", 2, 3, 2, [dag], seed=17)


# ---------------------------------------------------------------- P7 batching invariance
def test_batching_invariance():
    rng = np.random.default_rng(9)
    graphs = gen.make_graphs("sst_tree", 6, seed=9)
    h, d = 4, 3
    full = gen.batch_from_graphs(graphs, cell="tree_lstm", N=2, h=h, d=d, seed=9)
    ho_full, dp_full, dx_full, _ = oracle.run(full)
    perm = rng.permutation(len(graphs))
    dp_sum = np.zeros_like(dp_full)
    for k in perm:
        lo, hi = int(full.graph_ptr[k]), int(full.graph_ptr[k + 1])
        one = gen.batch_from_graphs([graphs[k]], cell="tree_lstm", N=2, h=h, d=d, seed=9,
                                    params=full.params)
        xr = full.x_row[lo:hi]
        one.x = full.x[xr[xr >= 0]]
        one.gamma = full.gamma[lo:hi]
        ho, dp, dx, _ = oracle.run(one)
        assert np.array_equal(ho, ho_full[lo:hi])
        dp_sum += dp
    np.testing.assert_allclose(dp_sum, dp_full, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- P9 bf16 emulation
def test_bf16_emulation_close_to_exact():
    b = gen.make_batch("tree_lstm", 2, 16, 16, "sst_tree", 6, seed=4)
    ho, dp, dx, _ = oracle.run(b)
    hq, dpq, dxq, _ = oracle.run(b, emulate_bf16=True)
    rel = lambda a, r: np.linalg.norm(a - r) / np.linalg.norm(r)
    assert 1e-5 < rel(hq, ho) < 2e-2
    assert rel(dpq, dp) < 2e-2
    assert rel(dxq, dx) < 2e-2
    # the default is Z11 (h~ rounded); the R-lin reading (exact sum of rounded slots) stays in the same band
    hr, dpr, dxr, _ = oracle.run(b, emulate_bf16=True, bf16_hsum="exact")
    assert 1e-5 < rel(hr, ho) < 2e-2
    assert rel(dpr, dp) < 2e-2


def test_bf16_fp32_accumulation_is_a_rounding_of_the_fp64_accumulation():
    """accum="fp32" (bf16 emulation): every product of bf16 operands is exact in fp32, so the
    fp32-accumulated emulation differs from the fp64-accumulated one only by the running sum's
    rounding -- on a contracting (well-conditioned) case by ~2^-24 * sqrt(K) relative, never more
    than a few 1e-6, and it does differ (the flag is live).  Without emulation it is the plain fp32
    evaluation: within ~1e-6 of fp64 on the same contracting case, and different from it."""
    b = gen.make_batch("tree_lstm", 2, 32, 32, "sst_tree", 6, seed=5)
    a = oracle.run(b, emulate_bf16=True)
    f = oracle.run(b, emulate_bf16=True, accum="fp32")
    rel = lambda x, r: np.linalg.norm(x - r) / np.linalg.norm(r)
    for x, y in zip(f[:3], a[:3]):
        assert rel(x, y) < 5e-6
    assert rel(f[0], a[0]) > 0
    e = oracle.run(b, accum="fp32")
    p = oracle.run(b)
    for x, y in zip(e[:3], p[:3]):
        assert rel(x, y) < 5e-6
    assert rel(e[0], p[0]) > 0


def test_bf16_hsum_readings_coincide_without_fan_in():
    """R-lin vs Z11: h~ = h_1 when no vertex has two children, and bf16 rounding is
    idempotent, so both readings must give bit-identical results on chains / unary trees."""
    b = gen.batch_from_graphs([[[], [0], [1], [], [3]], gen.chain(7)], cell="tree_lstm", N=2, h=8, d=8, seed=3,
                              x_at="all", loss_at="all")
    a = oracle.run(b, emulate_bf16=True, bf16_hsum="rounded")
    e = oracle.run(b, emulate_bf16=True, bf16_hsum="exact")
    for x, y in zip(a[:3], e[:3]):
        assert np.array_equal(x, y)


def test_bf16_hsum_rounded_is_a_bf16_rounding_of_the_exact_sum():
    """Z11's h~ is a bf16 number (low 16 bits of its fp32 image zero) within the bf16 unit
    roundoff 2^-8 of R-lin's exact sum of the rounded slots, at every vertex with >= 2 children;
    and the two readings do differ on binary trees (the flag is live)."""
    b = gen.make_batch("tree_lstm", 2, 16, 16, "sst_tree", 5, seed=8)
    _, ta = oracle.forward(b.cell, b.N, b.h, b.d, b.params, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, b.x,
                           emulate_bf16=True, bf16_hsum="rounded")
    _, te = oracle.forward(b.cell, b.N, b.h, b.d, b.params, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, b.x,
                           emulate_bf16=True, bf16_hsum="exact")
    differ = 0
    for v, ch in enumerate(ta.children):
        if len(ch) < 2:
            continue
        # compare at equal slot inputs: re-derive the exact sum from reading Z11's own rounded slots
        ex = sum(ta.st[v]["hkq"])
        hr = ta.st[v]["hs"]
        bits = np.asarray(hr, np.float32).view(np.uint32)
        assert np.all((bits & 0xFFFF) == 0)
        assert np.all(np.abs(hr - ex) <= 2.0 ** -8 * np.abs(ex) + 1e-300)
        differ += int(np.any(te.st[v]["hs"] != hr))
    assert differ > 0


# ---------------------------------------------------------------- NEXT-4 softmax head (outside (F, G))
def test_lm_head_matches_finite_differences_and_closed_forms():
    """The next-word head (reading Z9): dL/dh, dL/dW, dL/db against central differences of
    its own loss; with all-zero logits the per-row loss is log(vocab) (uniform softmax)."""
    rng = np.random.default_rng(3)
    V, h, vocab = 5, 3, 7
    H = rng.normal(size=(V, h))
    W = rng.normal(size=(vocab, h)) * 0.5
    b = rng.normal(size=vocab) * 0.1
    t = np.array([1, 6, -1, 0, 3])
    L, dH, dW, db = oracle.lm_head(H, W, b, t)
    eps = 1e-6
    for arr, grad in ((H, dH), (W, dW), (b, db)):
        num = np.zeros_like(arr)
        for j in np.ndindex(arr.shape):
            old = arr[j]
            arr[j] = old + eps; lp = oracle.lm_head(H, W, b, t)[0]
            arr[j] = old - eps; lm = oracle.lm_head(H, W, b, t)[0]
            arr[j] = old
            num[j] = (lp - lm) / (2 * eps)
        assert np.abs(num - grad).max() < 1e-7
    assert np.allclose(dH[2], 0) and np.allclose(oracle.lm_head(H, W * 0, b * 0, t)[0], 4 * np.log(vocab))

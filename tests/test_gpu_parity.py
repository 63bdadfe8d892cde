"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, on the same
seeded inputs.  Schedules bit-exact; fp32 mode within 1e-5 and bf16 mode within 2e-2
relative (BASELINE.json north_star), plus a tight check of the bf16 path against the
bf16-emulating oracle."""
import numpy as np
import pytest
import torch

import oracle
from oracle.cavs_oracle import global_children
from workloads import gen

from gpu_harness import compare, make_ctx, rel, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2
BF16_EMU_TOL = 5e-3   # bf16-emulating oracle has exact activations; the GPU uses MUFU tanh (2^-11)


def _sched_check(b, precision="fp32"):
    ctx = make_ctx(b, precision)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
    T = ctx.schedule()
    level, level_ptr, order = ctx.get_schedule()
    ch = global_children(b.graph_ptr, b.child_ptr, b.child_idx)
    rl, rlp, ro = oracle.schedule(ch)
    assert T == len(rlp) - 1
    assert np.array_equal(level, rl)
    assert np.array_equal(level_ptr, rlp)
    assert np.array_equal(order, ro)
    return T


# ------------------------------------------------------------------ schedule
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_schedule_bit_exact_configs(cfg):
    for seed in (0, 1):
        b = gen.make_config_batch(cfg, seed=seed, h=64) if cfg != "cfg5" else gen.make_config_batch(cfg, seed=seed, h=64)
        _sched_check(b)


@pytest.mark.parametrize("graphs", [
    "chain4096", "singletons", "forest", "star4", "mixed_spec", "deep_shallow"])
def test_schedule_adversarial(graphs):
    rng = np.random.default_rng(5)
    N = 2
    if graphs == "chain4096":
        g = [gen.permute(gen.chain(4096), rng), gen.chain(1)]
        N = 1
    elif graphs == "singletons":
        g = [[[]] for _ in range(37)]
    elif graphs == "forest":
        g = [[[], [], [0, 1], [], [3], [], [5]] for _ in range(5)]   # several roots per instance
    elif graphs == "star4":
        g = [[[1, 2, 3, 4], [], [], [], []]]
        N = 4
    elif graphs == "mixed_spec":
        g = [gen.chain(3), [[], [], [0, 1]]]
    else:
        g = [gen.permute(gen.chain(300), rng)] + [gen.permute(gen.remy_tree(5, rng), rng) for _ in range(50)]
        N = 2
    b = gen.batch_from_graphs(g, cell="tree_lstm", N=N, h=64, d=64, seed=1)
    _sched_check(b)


def test_schedule_mixed_batch_tasks():
    b = gen.batch_from_graphs([gen.chain(3), [[], [], [0, 1]]], cell="tree_lstm", N=2, h=64, d=64, seed=0)
    _sched_check(b)
    ctx = make_ctx(b, "fp32")
    ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    assert ctx.schedule() == 3
    _, lp, order = ctx.get_schedule()
    assert [sorted(order[lp[t]:lp[t + 1]].tolist()) for t in range(3)] == [[0, 3, 4], [1, 5], [2]]


# ------------------------------------------------------------------ errors
@pytest.mark.parametrize("graphs,N,code", [
    ([[[1], [0]]], 2, "E_CYCLE"),
    ([[[0]]], 2, "E_CYCLE"),
    ([[[], [0, 2], [1]]], 2, "E_CYCLE"),
    ([[[1, 2, 3], [], [], []]], 2, "E_ARITY"),
    ([[[5], []]], 2, "E_INVALID"),
    ([[[1, 2], [2], [0]]], 2, "E_CYCLE"),        # fan-out (DAG path) with a cycle
])
def test_schedule_errors(graphs, N, code):
    from paper_1712_04048_b200 import CavsError
    b = gen.batch_from_graphs(graphs, cell="tree_lstm", N=N, h=64, d=64, seed=0)
    ctx = make_ctx(b, "fp32", max_vertices=16, max_graphs=4, max_x=16)
    ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    with pytest.raises(CavsError) as e:
        ctx.schedule()
    assert e.value.name == code
    # a valid batch afterwards still works on the same context
    ok = gen.batch_from_graphs([gen.chain(2)], cell="tree_lstm", N=N, h=64, d=64, seed=0)
    ctx.load_graphs(ok.graph_ptr, ok.child_ptr, ok.child_idx)
    assert ctx.schedule() == 2


@pytest.mark.parametrize("graphs,N,code", [
    ([[[1], [0]]], 1, "E_CYCLE"),
    ([[[1, 2, 3], [], [], []]], 2, "E_ARITY"),
])
def test_deferred_schedule_errors_surface_at_forward(graphs, N, code):
    """schedule(wait=False) only enqueues; the validation error is returned by forward()."""
    from paper_1712_04048_b200 import CavsError
    dev = torch.device("cuda", 0)
    b = gen.batch_from_graphs(graphs, cell="tree_lstm", N=N, h=64, d=64, seed=0)
    ctx = make_ctx(b, "bf16", max_vertices=16, max_graphs=4, max_x=16)
    ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    assert ctx.schedule(wait=False) is None
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    with pytest.raises(CavsError) as e:
        ctx.forward(t(b.params), t(b.x), t(b.x_row))
    assert e.value.name == code


def test_deferred_schedule_matches_synchronous():
    b = BF16_CASES["tree_lstm_sst_h128_d64"]()
    g = run_gpu(b, "bf16")
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = make_ctx(b, "bf16")
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
    ctx.schedule(wait=False)
    h = ctx.forward(t(b.params), t(b.x), t(b.x_row))
    dp, dx = ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
    assert np.array_equal(h.cpu().numpy(), g["h_out"])
    assert np.array_equal(dp.cpu().numpy(), g["dparams"])
    assert np.array_equal(dx.cpu().numpy(), g["dx"])


def test_call_order_errors():
    from paper_1712_04048_b200 import CavsError
    b = gen.make_config_batch("cfg1", seed=0)
    ctx = make_ctx(b, "fp32")
    dev = torch.device("cuda", 0)
    with pytest.raises(CavsError) as e:
        ctx.schedule()
    assert e.value.name == "E_STATE"
    ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    ctx.schedule()
    with pytest.raises(CavsError) as e:
        ctx.backward(torch.zeros(b.V, b.h, device=dev), torch.zeros(ctx.P, device=dev), want_dx=False)
    assert e.value.name == "E_STATE"
    big = gen.make_config_batch("cfg1", seed=0, K=8)
    with pytest.raises(CavsError) as e:
        ctx.load_graphs(big.graph_ptr, big.child_ptr, big.child_idx)
    assert e.value.name == "E_CAPACITY"


# ------------------------------------------------------------------ fp32 numerics
FP32_CASES = {
    "cfg1_tree_fc": lambda: gen.make_config_batch("cfg1", seed=0),
    "cfg1_seed3": lambda: gen.make_config_batch("cfg1", seed=3),
    "tree_lstm_sst": lambda: gen.make_batch("tree_lstm", 2, 48, 40, "sst_tree", 24, seed=2),
    "lstm_chain": lambda: gen.make_batch("tree_lstm", 1, 40, 24, "sst_chain", 12, seed=3),
    "fixed_lstm": lambda: gen.make_batch("tree_lstm", 1, 32, 32, "chain64", 4, seed=4),
    "tree_fc_cbt": lambda: gen.make_batch("tree_fc", 2, 40, 24, "cbt32", 5, seed=5),
    "tree_lstm_N3": lambda: gen.batch_from_graphs(
        [[[], [], [], [0, 1, 2], [3], [], [4, 5]] for _ in range(3)] + [[[]]],
        cell="tree_lstm", N=3, h=24, d=16, seed=6, x_at="all", loss_at="all"),
    "tree_lstm_unary_forest": lambda: gen.batch_from_graphs(
        [[[], [], [0, 1], [], [3], [2, 4], [], [6]]] * 4, cell="tree_lstm", N=2, h=33, d=17, seed=7,
        x_at="all", loss_at="all"),
}


@pytest.mark.parametrize("case", list(FP32_CASES))
def test_fp32_parity(case):
    b = FP32_CASES[case]()
    g = run_gpu(b, "fp32")
    r = run_oracle(b)
    compare(b, g, r, FP32_TOL, case)


# FP32 mode on the tensor cores (h, d multiples of 64): bf16x3 split operands, six tcgen05 MMAs per
# product; the 1e-5 bar of the fp32 mode is unchanged
FP32_TC_CASES = {
    "lstm_sst_h64": lambda: gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 24, seed=81),
    "lstm_chain_h128": lambda: gen.make_batch("tree_lstm", 1, 128, 64, "sst_chain", 12, seed=82),
    "lstm_N3_h64": lambda: gen.batch_from_graphs(
        [[[], [], [], [0, 1, 2], [3], [], [4, 5]] for _ in range(5)] + [[[]]],
        cell="tree_lstm", N=3, h=64, d=64, seed=83, x_at="all", loss_at="all"),
    "fc_cbt_h128": lambda: gen.make_batch("tree_fc", 2, 128, 64, "cbt32", 5, seed=84),
    "lstm_sst_h256_d128": lambda: gen.make_batch("tree_lstm", 2, 256, 128, "sst_tree", 16, seed=85),
}


@pytest.mark.parametrize("case", list(FP32_TC_CASES))
def test_fp32_tensor_core_parity(case):
    """FP32 mode on tcgen05 against the fp64 oracle at the fp32 bar (1e-5), bit-reproducible."""
    b = FP32_TC_CASES[case]()
    g = run_gpu(b, "fp32")
    assert "bf16x3" in g["ctx"].path_info(), g["ctx"].path_info()
    compare(b, g, run_oracle(b), FP32_TOL, f"fp32 tcgen05 {case}")
    g2 = run_gpu(b, "fp32", ctx=g["ctx"])
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], g2[k]), f"{case}: {k} not deterministic"


def test_fp32_ffma_path_on_request(monkeypatch):
    """CAVS_FP32_FFMA=1 keeps the FFMA kernels; both fp32 engines agree with the oracle and with
    each other at the fp32 bar."""
    b = FP32_TC_CASES["lstm_sst_h64"]()
    monkeypatch.setenv("CAVS_FP32_FFMA", "1")
    f = run_gpu(b, "fp32")
    assert "FFMA" in f["ctx"].path_info(), f["ctx"].path_info()
    monkeypatch.delenv("CAVS_FP32_FFMA")
    t = run_gpu(b, "fp32")
    assert "bf16x3" in t["ctx"].path_info()
    compare(b, f, run_oracle(b), FP32_TOL, "fp32 FFMA vs fp64")
    compare(b, t, f, FP32_TOL, "fp32 tcgen05 vs FFMA")


def test_host_and_device_inputs_agree():
    b = gen.make_config_batch("cfg1", seed=1)
    g1 = run_gpu(b, "fp32", on_device=True)
    g2 = run_gpu(b, "fp32", on_device=False)
    assert np.array_equal(g1["h_out"], g2["h_out"])
    assert np.array_equal(g1["dparams"], g2["dparams"])


def test_context_reuse_across_batches():
    """Capacity sized for the largest batch; smaller/different batches reuse the arenas."""
    b0 = gen.make_batch("tree_lstm", 2, 32, 32, "sst_tree", 20, seed=8)
    b1 = gen.make_batch("tree_lstm", 2, 32, 32, "sst_tree", 7, seed=9)
    b1.params = b0.params
    ctx = make_ctx(b0, "fp32", max_vertices=b0.V + b1.V, max_graphs=40, max_x=b0.n_x + b1.n_x)
    for b in (b0, b1, b0):
        g = run_gpu(b, "fp32", ctx=ctx)
        compare(b, g, run_oracle(b), FP32_TOL, "reuse")


def test_train_step_host_matches_device_path():
    b = gen.make_batch("tree_lstm", 2, 32, 32, "sst_tree", 10, seed=10)
    g = run_gpu(b, "fp32")
    ctx = make_ctx(b, "fp32")
    dp = np.empty_like(b.params)
    dx = np.empty_like(b.x)
    ho = np.empty((b.V, b.h), np.float32)
    ctx.train_step_host(b.graph_ptr, b.child_ptr, b.child_idx, b.params, b.x, b.x_row, b.gamma, dp, dx, ho)
    assert np.array_equal(dp, g["dparams"])
    assert np.array_equal(dx, g["dx"])
    assert np.array_equal(ho, g["h_out"])


# ------------------------------------------------------------------ bf16 numerics
BF16_CASES = {
    "tree_lstm_sst_h64": lambda: gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 24, seed=11),
    "tree_lstm_sst_h128_d64": lambda: gen.make_batch("tree_lstm", 2, 128, 64, "sst_tree", 40, seed=12),
    "lstm_chain_h64": lambda: gen.make_batch("tree_lstm", 1, 64, 64, "sst_chain", 16, seed=13),
    "tree_fc_cbt_h64": lambda: gen.make_batch("tree_fc", 2, 64, 128, "cbt32", 6, seed=14),
    "tree_lstm_unary_h64": lambda: gen.batch_from_graphs(
        [[[], [], [0, 1], [], [3], [2, 4], [], [6]]] * 9, cell="tree_lstm", N=2, h=64, d=64, seed=15,
        x_at="all", loss_at="all"),
}


@pytest.mark.parametrize("case", list(BF16_CASES))
def test_bf16_parity(case):
    b = BF16_CASES[case]()
    g = run_gpu(b, "bf16")
    compare(b, g, run_oracle(b), BF16_TOL, case + " vs fp64 oracle")
    # diagnostics: the emulating oracle at the kernel's rounding points (R-lin) tightly, and at
    # SURVEY Z11's (h~ rounded) within the north_star gate
    compare(b, g, run_oracle(b, emulate_bf16=True, bf16_hsum="exact"), BF16_EMU_TOL,
            case + " vs bf16-emulating oracle (R-lin)")
    compare(b, g, run_oracle(b, emulate_bf16=True, bf16_hsum="rounded"), BF16_TOL,
            case + " vs bf16-emulating oracle (Z11)")


# ------------------------------------------------------------------ full-size (BASELINE sizes)
def _sub_batch(b, sample):
    """The graphs `sample` of b as their own batch (same params; x and Gamma rows carried over)."""
    from workloads.gen import subset_csr
    gp, cp, ci, rows, recs, nxr = subset_csr(b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, sample)
    sb = gen.Batch(cell=b.cell, N=b.N, h=b.h, d=b.d, graph_ptr=gp, child_ptr=cp, child_idx=ci, x_row=nxr,
                   x=b.x[recs], params=b.params, gamma=b.gamma[rows], is_chain=b.is_chain)
    return sb, rows, recs


def _clusters(ctx):
    """Graph-range clusters of the persistent level kernels (0 when the path is not persistent)."""
    import re
    m = re.search(r"(\d+) clusters of", ctx.path_info())
    return int(m.group(1)) if m else 0


def _cluster_sample(b, ncl):
    """One graph per persistent-kernel cluster (the deepest of its range: cl(g) = graph_ptr[g]·R/V,
    sched.cu k_level_offsets), so every cluster's backward is exercised; two graphs otherwise."""
    lv = oracle.levels_recursive(global_children(b.graph_ptr, b.child_ptr, b.child_idx))
    depth = [int(lv[b.graph_ptr[k]:b.graph_ptr[k + 1]].max()) for k in range(b.K)]
    if ncl <= 0:
        return sorted({int(np.argmax(depth)), b.K - 1})
    best = {}
    for k in range(b.K):
        c = int(int(b.graph_ptr[k]) * ncl // b.V)
        if c not in best or depth[k] > depth[best[c]]:
            best[c] = k
    return sorted(best.values())


def _quant(q, r, b):
    """bf16 quantisation of a workload: emulating oracle vs fp64 oracle, worst tensor."""
    from gpu_harness import param_blocks
    return max([rel(q["h_out"], r["h_out"]), rel(q["dx"], r["dx"])] +
               [rel(q["dparams"][sl], r["dparams"][sl]) for _, sl in param_blocks(b)])


@pytest.mark.parametrize("cfg,precision", [("cfg4", "bf16"), ("cfg4", "fp32")])
def test_full_size_cfg4_all_graphs(cfg, precision):
    """BASELINE cfg4 (256 SST-shaped trees, h = 512) in the bench's launch configuration.
    Forward: h_out of ALL 256 graphs against the fp64 oracle, row by row.  Backward: Gamma kept
    on one graph per persistent-kernel cluster (every cluster's backward runs), so the full-batch
    dparams / dx equal the oracle's over that sample (graphs are independent)."""
    b = gen.make_config_batch(cfg, seed=0)
    tol = FP32_TOL if precision == "fp32" else BF16_TOL
    ctx = make_ctx(b, "bf16")
    sample = _cluster_sample(b, _clusters(ctx))
    ctx.close()
    keep = np.zeros(b.V, bool)
    for k in sample:
        keep[b.graph_ptr[k]:b.graph_ptr[k + 1]] = True
    b.gamma[~keep] = 0
    g = run_gpu(b, precision)
    ho, _ = oracle.forward(b.cell, b.N, b.h, b.d, b.params, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, b.x)
    from gpu_harness import row_rel_max, elem_rel_max, RECORD
    e = {"h_out": rel(g["h_out"], ho), "h_out.row": row_rel_max(g["h_out"], ho), "h_out.elem": elem_rel_max(g["h_out"], ho)}
    RECORD.append({"what": f"{cfg} {precision} all 256 graphs h_out vs fp64", "tol": tol, "errs": e})
    assert e["h_out"] <= tol and e["h_out.row"] <= 5 * tol and e["h_out.elem"] <= 2 * tol, e
    sb, rows, recs = _sub_batch(b, sample)
    r = run_oracle(sb)
    g_s = dict(h_out=g["h_out"][rows], dparams=g["dparams"], dx=g["dx"][recs])
    compare(b, g_s, r, tol, f"{cfg} {precision} backward sample {sample} vs fp64")
    if precision == "bf16":
        q = run_oracle(sb, emulate_bf16=True, bf16_hsum="exact")
        assert _quant(q, r, b) <= 1e-2          # the fp64 2e-2 gate above is meaningful for this workload
        compare(b, g_s, q, 2 * BF16_EMU_TOL, f"{cfg} bf16 backward sample vs bf16-emulating oracle (R-lin)")


@pytest.mark.parametrize("cfg,precision,sample", [
    ("cfg2", "bf16", [5, 63]), ("cfg3", "bf16", [17, 200]), ("cfg4_h1024", "bf16", [31, 255]),
    ("cfg2", "fp32", [7]), ("cfg3", "fp32", [200])])
def test_full_size_sampled(cfg, precision, sample):
    """BASELINE sizes in the bench's launch configuration; Gamma zeroed outside the sampled graphs,
    whose h rows, dparams and dx are checked against the fp64 oracle, unconditionally at the
    north_star tolerance, and (bf16) against the bf16-emulating oracle."""
    b = gen.make_config_batch(cfg, seed=0)
    keep = np.zeros(b.V, bool)
    for k in sample:
        keep[b.graph_ptr[k]:b.graph_ptr[k + 1]] = True
    b.gamma[~keep] = 0
    g = run_gpu(b, precision)
    sb, rows, recs = _sub_batch(b, sample)
    r = run_oracle(sb)
    g_s = dict(h_out=g["h_out"][rows], dparams=g["dparams"], dx=g["dx"][recs])
    compare(b, g_s, r, FP32_TOL if precision == "fp32" else BF16_TOL, f"{cfg} {precision} sample {sample} vs fp64")
    if precision == "bf16":
        q = run_oracle(sb, emulate_bf16=True, bf16_hsum="exact")
        assert _quant(q, r, b) <= 1e-2
        compare(b, g_s, q, 2 * BF16_EMU_TOL, f"{cfg} bf16 sample vs bf16-emulating oracle (R-lin)")


@pytest.mark.parametrize("precision,pscale", [("bf16", 1.0), ("fp32", 1.0), ("bf16", 0.1)])
def test_full_size_cfg5(precision, pscale):
    """cfg5 (Tree-FC CBT-256, h = 2048, 64 graphs) at the bench's OWN init (pscale 1) and with a
    contracting init (pscale 0.1).  At the bench init F is chaotic (reading R-chaos): bf16 operand
    rounding alone moves dW by ~20% against fp64 and fp32 rounding moves it by ~1e-4, so there the
    GPU is gated by the conditioning-derived band (below); the contracting init is gated at the
    precision's tolerance against fp64 (and bf16 also against the emulating oracle)."""
    b = gen.make_config_batch("cfg5", seed=0)
    b.params = (b.params * pscale).astype(np.float32)
    sample = [9, 40]
    keep = np.zeros(b.V, bool)
    for k in sample:
        keep[b.graph_ptr[k]:b.graph_ptr[k + 1]] = True
    b.gamma[~keep] = 0
    g = run_gpu(b, precision)
    sb, rows, recs = _sub_batch(b, sample)
    g_s = dict(h_out=g["h_out"][rows], dparams=g["dparams"], dx=g["dx"][recs])
    emu = precision == "bf16"
    tol = BF16_TOL if emu else FP32_TOL
    if pscale == 1.0:
        # chaotic F (reading R-chaos): any change of rounding -- fp32 summation order, the MUFU
        # tanh -- is amplified by the dynamics, in fp32 as in bf16.  The band is the problem's own
        # conditioning: the distance between two equally valid evaluations (fp64- vs fp32-computed
        # products, same rounding points otherwise), times 4 (the GPU's activations perturb more
        # than the products' rounding does), never tighter than the precision's gate.
        q = run_oracle(sb, emulate_bf16=emu)
        q32 = run_oracle(sb, emulate_bf16=emu, accum="fp32")
        from gpu_harness import errors, RECORD
        spread = errors(b, q32, q)
        g_err = errors(b, g_s, q)
        RECORD.append({"what": f"cfg5 {precision} bench init: evaluation spread (fp32 vs fp64 products)",
                       "tol": None, "errs": spread})
        RECORD.append({"what": f"cfg5 {precision} bench init vs oracle", "tol": None, "errs": g_err})
        bad = {k: (v, spread[k]) for k, v in g_err.items() if not v <= max(tol, 4 * spread[k])}
        assert not bad, f"cfg5 bench init: GPU vs oracle beyond 4x the evaluation spread: {bad}"
        assert max(spread.values()) > tol, "R-chaos: the bench init should be ill-conditioned"
        return
    if precision == "fp32":
        compare(b, g_s, run_oracle(sb), FP32_TOL, f"cfg5 fp32 x{pscale} vs fp64")
        return
    q = run_oracle(sb, emulate_bf16=True)
    r = run_oracle(sb)
    assert _quant(q, r, b) <= 1e-2
    compare(b, g_s, r, BF16_TOL, f"cfg5 bf16 x{pscale} vs fp64")
    compare(b, g_s, q, 2 * BF16_EMU_TOL, f"cfg5 bf16 x{pscale} vs bf16-emulating oracle")


@pytest.mark.parametrize("case", ["tree_lstm_sst_h128_d64", "lstm_chain_h64", "tree_fc_cbt_h64"])
def test_tcgen05_matches_simt_bf16(case, monkeypatch):
    """Same bf16 rounding points on both paths; only the accumulation order differs."""
    b = BF16_CASES[case]()
    monkeypatch.setenv("CAVS_BF16_SIMT", "1")
    s = run_gpu(b, "bf16")
    monkeypatch.setenv("CAVS_BF16_SIMT", "0")
    t = run_gpu(b, "bf16")
    from gpu_harness import compare
    compare(b, t, s, BF16_EMU_TOL, case + " tcgen05 vs simt-bf16")


@pytest.mark.parametrize("case", ["tree_lstm_sst_h128_d64", "lstm_chain_h64", "tree_fc_cbt_h64", "tree_lstm_unary_h64"])
def test_gate_split_cluster_matches_monolithic(case, monkeypatch):
    """The 4-CTA gate-split cluster kernels against the one-CTA-per-unit-block kernels:
    identical operands and rounding points, different fp32 summation order only."""
    b = BF16_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "0")
    monkeypatch.setenv("CAVS_TC_MONO", "1")
    m = run_gpu(b, "bf16")
    monkeypatch.setenv("CAVS_TC_MONO", "0")
    g = run_gpu(b, "bf16")
    from gpu_harness import compare
    compare(b, g, m, 1e-3, case + " gate-split vs monolithic")


# ------------------------------------------------------------------ persistent level kernel
def _nary_forest(K, N, max_leaves, seed):
    """Random trees whose internal vertices have 1..N children (children before parents)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(K):
        nodes = [[] for _ in range(int(rng.integers(1, max_leaves + 1)))]
        frontier = list(range(len(nodes)))
        while len(frontier) > 1:
            k = int(rng.integers(1, min(N, len(frontier)) + 1))
            pick = sorted(rng.choice(len(frontier), size=k, replace=False).tolist(), reverse=True)
            ch = [frontier.pop(i) for i in pick]
            nodes.append(ch)
            frontier.append(len(nodes) - 1)
        out.append(gen.permute(nodes, rng))
    return out


PERSIST_CASES = {
    # h = 512: 16 unit blocks x 9 replicas; NT = 16/32/64 across the levels
    "lstm_n2_h512_sst": lambda: gen.make_batch("tree_lstm", 2, 512, 512, "sst_tree", 40, seed=21),
    # h = 256, 2 rounds of NT = 64 tiles per task (600 chains of 3 > 64 x 18 replicas / 2)
    "lstm_n1_h256_wide": lambda: gen.batch_from_graphs([gen.chain(3)] * 1300, cell="tree_lstm", N=1, h=256, d=128,
                                                        seed=22, x_at="all", loss_at="all"),
    # 300 tasks in one launch: 299 grid barriers
    "lstm_n1_h64_deep": lambda: gen.batch_from_graphs([gen.chain(300), gen.chain(120)], cell="tree_lstm", N=1,
                                                       h=64, d=64, seed=23, x_at="all", loss_at="all"),
    "lstm_n3_h128": lambda: gen.batch_from_graphs(_nary_forest(30, 3, 20, 24), cell="tree_lstm", N=3, h=128, d=64,
                                                  seed=24),
    "lstm_n4_h512": lambda: gen.batch_from_graphs(_nary_forest(12, 4, 24, 25), cell="tree_lstm", N=4, h=512, d=128,
                                                  seed=25),
    # h = 384: 3 unit blocks x 4 K-slices of unequal width (iou 4/5/4/5, U_f 1/2/1/2 k-blocks)
    "lstm_n2_h384_sst": lambda: gen.make_batch("tree_lstm", 2, 384, 256, "sst_tree", 30, seed=29),
    "lstm_unary_h128": lambda: gen.batch_from_graphs(
        [[[], [], [0, 1], [], [3], [2, 4], [], [6]]] * 9, cell="tree_lstm", N=2, h=128, d=64, seed=26,
        x_at="all", loss_at="all"),
    "fc_h256_cbt": lambda: gen.make_batch("tree_fc", 2, 256, 128, "cbt32", 12, seed=27),
    "fc_h512_sst": lambda: gen.make_batch("tree_fc", 2, 512, 256, "sst_tree", 24, seed=28),
}


@pytest.mark.parametrize("case", list(PERSIST_CASES))
def test_persistent_levels(case, monkeypatch):
    """One persistent weight-stationary launch per pass (persist.cu) against the oracle, and
    against the per-task launches (CAVS_PERSIST=0: same operands and rounding points)."""
    b = PERSIST_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "1")
    g = run_gpu(b, "bf16")
    assert "levels: persistent" in g["ctx"].path_info(), g["ctx"].path_info()
    compare(b, g, run_oracle(b), BF16_TOL, case + " vs fp64 oracle")
    # deep / wide trees: single-ulp bf16 rounding flips of h (different fp32 summation order than
    # the emulating oracle's) accumulate in the weight gradients; still 2x inside the 2e-2 gate
    compare(b, g, run_oracle(b, emulate_bf16=True, bf16_hsum="exact"), 2 * BF16_EMU_TOL,
            case + " vs bf16-emulating oracle (R-lin)")
    monkeypatch.setenv("CAVS_PERSIST", "0")
    o = run_gpu(b, "bf16")
    assert "levels: persistent" not in o["ctx"].path_info()
    # the per-task path (split-K row kernels, K-sliced clusters) sums in yet another fp32 order: the
    # same deep / wide-tree allowance as against the emulating oracle (fc_h512_sst: db 5.0e-3)
    compare(b, g, o, 2 * BF16_EMU_TOL, case + " persistent vs per-task")


KSPLIT_CASES = ["lstm_n2_h512_sst", "lstm_n1_h256_wide", "lstm_n3_h128", "lstm_n4_h512", "lstm_n2_h384_sst",
                "lstm_unary_h128"]


@pytest.mark.parametrize("case", KSPLIT_CASES)
def test_ksplit_backward(case, monkeypatch):
    """The opt-in K-split Tree-LSTM backward (CAVS_PBWD=1, persist_bwd.cu: 4 K-slices per 128-unit
    block, partials reduced over DSMEM in fixed order) against the default gate-grouped backward:
    same bf16 operands and rounding points, another fp32 summation order; bit-identical when the
    same context runs the same batch twice."""
    b = PERSIST_CASES[case]()
    monkeypatch.setenv("CAVS_PBWD", "1")
    g = run_gpu(b, "bf16")
    assert "bwd K-split" in g["ctx"].path_info(), g["ctx"].path_info()
    g2 = run_gpu(b, "bf16", ctx=g["ctx"])
    assert np.array_equal(g["dparams"], g2["dparams"]) and np.array_equal(g["dx"], g2["dx"]), \
        "K-split backward not deterministic"
    monkeypatch.delenv("CAVS_PBWD")
    o = run_gpu(b, "bf16")
    assert "bwd K-split" not in o["ctx"].path_info()
    assert np.array_equal(g["h_out"], o["h_out"])          # same forward kernel
    compare(b, g, o, BF16_EMU_TOL, case + " K-split vs gate-grouped backward")


def test_persistent_path_is_default_for_benchmark_shape():
    b = gen.make_batch("tree_lstm", 2, 512, 512, "sst_tree", 4, seed=1)
    ctx = make_ctx(b, "bf16")
    assert "levels: persistent" in ctx.path_info() and "bwd gate-grouped" in ctx.path_info(), ctx.path_info()


# ------------------------------------------------------------------ stream-K lazy gradients
LAZY_CASES = {
    "lstm_n2_h512_sst": lambda: gen.make_batch("tree_lstm", 2, 512, 512, "sst_tree", 40, seed=31),
    "lstm_n1_h256_chain": lambda: gen.batch_from_graphs([gen.chain(n) for n in (40, 17, 3, 60)], cell="tree_lstm",
                                                         N=1, h=256, d=128, seed=32, x_at="all", loss_at="all"),
    "lstm_n3_h128": lambda: gen.batch_from_graphs(_nary_forest(30, 3, 20, 33), cell="tree_lstm", N=3, h=128, d=192,
                                                  seed=33),
    # no internal vertex: every dU tile is a zero-work piece
    "lstm_leaves_only": lambda: gen.batch_from_graphs([[[]]] * 70, cell="tree_lstm", N=2, h=128, d=64, seed=34,
                                                      loss_at="all"),
    # no pull record: every dW tile is a zero-work piece
    "lstm_no_x": lambda: gen.batch_from_graphs(_nary_forest(20, 2, 12, 35), cell="tree_lstm", N=2, h=128, d=64,
                                               seed=35, x_at="none"),
    "fc_h256_cbt": lambda: gen.make_batch("tree_fc", 2, 256, 128, "cbt32", 12, seed=36),
    "fc_h512_sst": lambda: gen.make_batch("tree_fc", 2, 512, 256, "sst_tree", 60, seed=37),
}


@pytest.mark.parametrize("case", list(LAZY_CASES))
def test_lazy_streamk(case, monkeypatch):
    """The one-launch stream-K lazy kernel (lazy.cu) against the oracle and against the split-K
    type-II kernels + pack (CAVS_LAZY=0): same bf16 operands, fp32 sums in another order; and
    bit-identical results when the same context runs the same batch twice (fixed-order in-kernel
    split-K reduction)."""
    b = LAZY_CASES[case]()
    monkeypatch.setenv("CAVS_LAZY", "1")
    g = run_gpu(b, "bf16")
    assert "lazy: stream-K" in g["ctx"].path_info(), g["ctx"].path_info()
    compare(b, g, run_oracle(b), BF16_TOL, case + " vs fp64 oracle")
    g2 = run_gpu(b, "bf16", ctx=g["ctx"])
    assert np.array_equal(g["dparams"], g2["dparams"]), "stream-K lazy gradients not deterministic"
    monkeypatch.setenv("CAVS_LAZY", "0")
    o = run_gpu(b, "bf16")
    assert "lazy: split-K" in o["ctx"].path_info()
    compare(b, g, o, 1e-5, case + " stream-K vs split-K")


# ------------------------------------------------------------------ row-tiled large-task kernels
ROWS_CASES = {
    "lstm_n2_h256_sst": lambda: gen.make_batch("tree_lstm", 2, 256, 128, "sst_tree", 48, seed=41),
    "lstm_n1_h128_chain": lambda: gen.batch_from_graphs([gen.chain(n) for n in (30, 200, 7)] * 60, cell="tree_lstm",
                                                         N=1, h=128, d=128, seed=42, x_at="all", loss_at="all"),
    "lstm_n2_h128_unary": lambda: gen.batch_from_graphs(_nary_forest(60, 2, 30, 43), cell="tree_lstm", N=2, h=128,
                                                        d=64, seed=43),
    "fc_h256_cbt": lambda: gen.make_batch("tree_fc", 2, 256, 128, "cbt32", 40, seed=44),
    "fc_h512_sst": lambda: gen.make_batch("tree_fc", 2, 512, 256, "sst_tree", 60, seed=45),
}


@pytest.mark.parametrize("case", list(ROWS_CASES))
def test_rows_level_kernels(case, monkeypatch):
    """Row-tiled tcgen05 level GEMMs (rows.cu; forced onto every non-skinny task) against the oracle
    and against the per-task swap-AB kernels (CAVS_ROWS=0): same bf16 operands and rounding
    points, another fp32 summation order."""
    b = ROWS_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "0")
    monkeypatch.setenv("CAVS_ROWS_MIN_TILES", "1")
    g = run_gpu(b, "bf16")
    assert "large tasks: row-tiled" in g["ctx"].path_info(), g["ctx"].path_info()
    compare(b, g, run_oracle(b), BF16_TOL, case + " vs fp64 oracle")
    compare(b, g, run_oracle(b, emulate_bf16=True, bf16_hsum="exact"), 2 * BF16_EMU_TOL,
            case + " vs bf16-emulating oracle (R-lin)")
    monkeypatch.setenv("CAVS_ROWS", "0")
    o = run_gpu(b, "bf16")
    assert "row-tiled" not in o["ctx"].path_info()
    compare(b, g, o, BF16_EMU_TOL, case + " row-tiled vs per-task")


@pytest.mark.parametrize("case", ["fc_h256_cbt", "lstm_n2_h256_sst", "lstm_n1_h128_chain"])
def test_rows_split_k(case, monkeypatch):
    """Split-K of the row-tiled kernel (tasks whose tiles leave SMs idle: K shares, fp32 partials summed
    in share order by the last share to arrive): against the oracle, bit-reproducible, and against the
    unsplit kernel (CAVS_ROWS_KSPLIT=0: same bf16 operands, another fp32 summation order)."""
    b = ROWS_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "0")
    monkeypatch.setenv("CAVS_ROWS_MIN_TILES", "1")
    g = run_gpu(b, "bf16")
    compare(b, g, run_oracle(b), BF16_TOL, case + " split-K vs fp64 oracle")
    g2 = run_gpu(b, "bf16", ctx=g["ctx"])
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], g2[k]), f"{case}: split-K {k} not deterministic"
    monkeypatch.setenv("CAVS_ROWS_DSM", "1")               # partials exchanged through DSMEM (opt-in)
    q = run_gpu(b, "bf16")
    for k in ("h_out", "dparams", "dx"):                   # same partials, same share order
        assert np.array_equal(g[k], q[k]), f"{case}: DSMEM vs global split-K {k} differ"
    monkeypatch.delenv("CAVS_ROWS_DSM")
    monkeypatch.setenv("CAVS_ROWS_KSPLIT", "0")
    o = run_gpu(b, "bf16")
    compare(b, g, o, BF16_EMU_TOL, case + " split-K vs unsplit")


KSL_CASES = {
    "lstm_n2_h128_sst": lambda: gen.make_batch("tree_lstm", 2, 128, 64, "sst_tree", 10, seed=91),
    "lstm_n1_h256_chain": lambda: gen.batch_from_graphs([gen.chain(n) for n in (9, 30, 2, 17)], cell="tree_lstm", N=1,
                                                        h=256, d=128, seed=92, x_at="all", loss_at="all"),
    "fc_h256_cbt": lambda: gen.make_batch("tree_fc", 2, 256, 128, "cbt16", 6, seed=93),
}


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("ksl", ["2", "4"])
@pytest.mark.parametrize("case", list(KSL_CASES))
def test_ksliced_gate_split(case, ksl, precision, monkeypatch):
    """Per-task kernels with K-sliced gate-split clusters (4 x ksl CTAs per 128-unit block, the slices'
    accumulators summed through DSMEM like the gate ranks) against the oracle, bit-reproducible, and
    against the plain gate split (same operands, another fp32 summation order)."""
    b = KSL_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "0")
    monkeypatch.setenv("CAVS_ROWS", "0")
    monkeypatch.setenv("CAVS_TC_KSL", ksl)
    g = run_gpu(b, precision)
    tol = FP32_TOL if precision == "fp32" else BF16_TOL
    compare(b, g, run_oracle(b), tol, f"ksl {ksl} {case} {precision} vs fp64")
    g2 = run_gpu(b, precision, ctx=g["ctx"])
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], g2[k]), f"{case}: {k} not deterministic"
    monkeypatch.setenv("CAVS_TC_KSL", "1")
    o = run_gpu(b, precision)
    compare(b, g, o, FP32_TOL if precision == "fp32" else BF16_EMU_TOL, f"ksl {ksl} vs 1 {case} {precision}")


XD_CASES = {   # d % 256 == 0: dX tiles of 256 input columns
    "lstm_n2_h256_d256_sst": lambda: gen.make_batch("tree_lstm", 2, 256, 256, "sst_tree", 24, seed=95),
    "lstm_n1_h128_d256_chain": lambda: gen.batch_from_graphs([gen.chain(n) for n in (30, 200, 7)] * 20,
                                                             cell="tree_lstm", N=1, h=128, d=256, seed=96, x_at="all",
                                                             loss_at="all"),
    "fc_h256_d256_cbt": lambda: gen.make_batch("tree_fc", 2, 256, 256, "cbt32", 20, seed=97),
    "fc_h512_sst": lambda: ROWS_CASES["fc_h512_sst"](),
}


@pytest.mark.parametrize("case", list(XD_CASES))
def test_rows_xproj_dx(case, monkeypatch):
    """The eager x-projection and dX on the row-tiled kernel (row tiles without an epilogue row skipped)
    against the oracle and against the row GEMMs of gemm.cu (CAVS_ROWS_XD=0: same bf16 operands, another
    fp32 summation order); bit-reproducible."""
    b = XD_CASES[case]()
    monkeypatch.setenv("CAVS_ROWS_XD", "1")               # (default on for Tree-FC, opt-in for Tree-LSTM)
    g = run_gpu(b, "bf16")
    assert "x-projection / dX: row-tiled" in g["ctx"].path_info(), g["ctx"].path_info()
    compare(b, g, run_oracle(b), BF16_TOL, case + " rows x-projection / dX vs fp64 oracle")
    g2 = run_gpu(b, "bf16", ctx=g["ctx"])
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], g2[k]), f"{case}: {k} not deterministic"
    monkeypatch.setenv("CAVS_ROWS_XD", "0")
    o = run_gpu(b, "bf16")
    assert "x-projection / dX: row-tiled" not in o["ctx"].path_info()
    compare(b, g, o, 2 * BF16_EMU_TOL, case + " rows vs gemm_rows x-projection / dX")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("case", ["lstm_n2_h128_sst", "fc_h256_cbt"])
def test_grouped_stages(case, precision, monkeypatch):
    """Opt-in grouped pipeline stages of the per-task kernels (CAVS_TC_GROUP=1: 4-D TMA boxes over k-blocks
    and planes) against the per-k-block boxes: same operands, same summation order -> bit-identical."""
    b = KSL_CASES[case]()
    monkeypatch.setenv("CAVS_PERSIST", "0")
    monkeypatch.setenv("CAVS_ROWS", "0")
    o = run_gpu(b, precision)
    monkeypatch.setenv("CAVS_TC_GROUP", "1")
    g = run_gpu(b, precision)
    compare(b, g, run_oracle(b), FP32_TOL if precision == "fp32" else BF16_TOL, f"grouped {case} {precision}")
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], o[k]), f"{case} {precision}: grouped stages change {k}"


# ------------------------------------------------------------------ inference-only forward
@pytest.mark.parametrize("case", ["lstm_n2_h512_sst", "fc_h256_cbt"])
@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_forward_inference(case, precision, monkeypatch):
    """cavs_forward_inference: the same h_out as the training forward, bit for bit (the same
    kernels minus the activation stores), and a backward right after it is a usage error."""
    from paper_1712_04048_b200 import CavsError
    b = LAZY_CASES[case]() if case in LAZY_CASES else PERSIST_CASES[case]()
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = make_ctx(b, precision)
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
    ctx.schedule()
    h_inf = ctx.forward_inference(t(b.params), t(b.x), t(b.x_row)).cpu().numpy()
    with pytest.raises(CavsError):
        ctx.backward(t(b.gamma))
    h_trn = ctx.forward(t(b.params), t(b.x), t(b.x_row)).cpu().numpy()
    assert np.array_equal(h_inf, h_trn)
    ref = run_oracle(b)
    assert rel(h_inf, ref["h_out"]) <= (FP32_TOL if precision == "fp32" else BF16_TOL)
    dp, _ = ctx.backward(t(b.gamma))                  # a training forward re-enables backward
    torch.cuda.synchronize()


# ------------------------------------------------------------------ pull records: sharing, range
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_shared_pull_records_accumulate_dx(precision):
    """Several vertices pulling the same record (an embedding row, P:L606's word inputs): dx of
    the record is the SUM of their pull adjoints; an unreferenced record gets 0."""
    b = gen.make_batch("tree_lstm", 1, 64, 64, "sst_chain", 12, seed=51)
    rng = np.random.default_rng(51)
    n_rec = 23                                       # 23 + 1 unreferenced records for ~230 vertices
    b.x_row = rng.integers(0, n_rec, size=b.V).astype(np.int32)
    b.x = np.random.default_rng(52).uniform(-1, 1, size=(n_rec + 1, b.d)).astype(np.float32)
    g = run_gpu(b, precision)
    assert np.all(g["dx"][n_rec] == 0)
    compare(b, g, run_oracle(b), FP32_TOL if precision == "fp32" else BF16_TOL, f"shared records {precision}")


def test_out_of_range_x_row_is_a_deferred_error():
    from paper_1712_04048_b200 import CavsError
    b = gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 4, seed=53)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = make_ctx(b, "bf16")
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
    ctx.schedule()
    xr = b.x_row.copy()
    xr[0] = b.n_x + 5
    ctx.forward(t(b.params), t(b.x), t(xr))
    with pytest.raises(CavsError) as e:
        ctx.sync()
    assert e.value.name == "E_INVALID"
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))   # a new schedule clears it
    ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row))
    ctx.sync()


# ------------------------------------------------------------------ DAG inputs (NEXT-3)
def _random_dags(K, N, n_max, seed, tree_frac=0.0):
    """Random DAGs: vertices are created children-first; an internal vertex lists 1..N children drawn
    WITH replacement from all earlier vertices (fan-out and duplicate child ids), local ids permuted.
    A fraction of the graphs are plain trees (a batch mixing both runs the DAG path)."""
    rng = np.random.default_rng(seed)
    out = []
    for g in range(K):
        if rng.random() < tree_frac:
            out.append(_nary_forest(1, N, int(rng.integers(1, n_max // 2 + 1)), int(rng.integers(1 << 30)))[0])
            continue
        n = int(rng.integers(1, n_max + 1))
        nodes = []
        for v in range(n):
            if v < 2 or rng.random() < 0.3:
                nodes.append([])
            else:
                k = int(rng.integers(1, N + 1))
                nodes.append(rng.integers(0, v, size=k).tolist())
        out.append(gen.permute(nodes, rng))
    return out


DAG_CASES = {
    "lstm_n2_h64": lambda: gen.batch_from_graphs(_random_dags(20, 2, 30, 51), cell="tree_lstm", N=2, h=64, d=64,
                                                 seed=51, x_at="all", loss_at="all"),
    "lstm_n3_h128_mixed": lambda: gen.batch_from_graphs(_random_dags(24, 3, 40, 52, tree_frac=0.5), cell="tree_lstm",
                                                        N=3, h=128, d=64, seed=52, x_at="all", loss_at="all"),
    "lstm_n2_h512": lambda: gen.batch_from_graphs(_random_dags(30, 2, 60, 53), cell="tree_lstm", N=2, h=512,
                                                  d=512, seed=53, x_at="all", loss_at="all"),
    "fc_h128": lambda: gen.batch_from_graphs(_random_dags(20, 2, 40, 54), cell="tree_fc", N=2, h=128, d=64,
                                             seed=54, x_at="all", loss_at="all"),
}


@pytest.mark.parametrize("case", list(DAG_CASES))
def test_dag_schedule_bit_exact(case):
    b = DAG_CASES[case]()
    ctx = make_ctx(b, "bf16")
    ctx.load_graphs(b.graph_ptr, b.child_ptr, b.child_idx)
    T = ctx.schedule()
    level, lp, order = ctx.get_schedule()
    ch = global_children(b.graph_ptr, b.child_ptr, b.child_idx)
    lv, lp_r, order_r = oracle.schedule(ch)
    assert T == len(lp_r) - 1
    assert np.array_equal(level, lv) and np.array_equal(lp, lp_r) and np.array_equal(order, order_r)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("case", list(DAG_CASES))
def test_dag_parity(case, precision):
    """DAG batches (fan-out, duplicate child ids, trees mixed in) against the fp64 oracle, whose
    additive backward is pinned by finite differences on DAGs (test_oracle_pins); bit-identical
    when run twice (fixed-order pull-reduce over the parent CSR)."""
    b = DAG_CASES[case]()
    g = run_gpu(b, precision)
    r = run_oracle(b)
    compare(b, g, r, FP32_TOL if precision == "fp32" else BF16_TOL, f"DAG {case} {precision} vs fp64")
    g2 = run_gpu(b, precision, ctx=g["ctx"])
    for k in ("h_out", "dparams", "dx"):
        assert np.array_equal(g[k], g2[k]), f"DAG {case}: {k} not deterministic"
    # a tree batch on the same context afterwards still takes the fused tree path
    t = gen.make_batch(b.cell, b.N, b.h, b.d, "sst_tree" if b.cell == "tree_lstm" else "cbt8", 3, seed=5)
    gt = run_gpu(t, precision, ctx=g["ctx"])
    compare(t, gt, run_oracle(t), FP32_TOL if precision == "fp32" else BF16_TOL, f"tree after DAG {case}")


# ------------------------------------------------------------------ engine ablations (NEXT-1)
ABLATIONS = {
    "lazy_off": ({"CAVS_LAZY_BATCH": "0"}, "lazy batching OFF"),
    "unfused": ({"CAVS_UNFUSED": "1"}, "unfused cell epilogues"),
    "streaming": ({"CAVS_STREAMING": "1"}, "streamed x-projection"),
}
ABL_CASES = {
    "lstm_sst_h128": lambda: gen.make_batch("tree_lstm", 2, 128, 128, "sst_tree", 12, seed=61),
    "lstm_chains_h64": lambda: gen.batch_from_graphs([gen.chain(n) for n in (9, 30, 2, 17)], cell="tree_lstm", N=1,
                                                     h=64, d=64, seed=62, x_at="all", loss_at="all"),
    "fc_cbt_h128": lambda: gen.make_batch("tree_fc", 2, 128, 64, "cbt16", 6, seed=63),
    "lstm_dag_h64": lambda: DAG_CASES["lstm_n2_h64"](),
}


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("case", list(ABL_CASES))
@pytest.mark.parametrize("abl", list(ABLATIONS))
def test_ablations(abl, case, precision, monkeypatch):
    """The paper's optimisation toggles (Fig. 10; lazy batching P:L542, fusion P:L559-562,
    streaming P:L544) change where and when the same arithmetic runs, not the method: each ablated
    engine against the fp64 oracle, and against the default engine (same operands and rounding
    points; only fp32 summation order may differ)."""
    b = ABL_CASES[case]()
    env, marker = ABLATIONS[abl]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = run_gpu(b, precision)
    assert marker in g["ctx"].path_info(), g["ctx"].path_info()
    tol = FP32_TOL if precision == "fp32" else BF16_TOL
    compare(b, g, run_oracle(b), tol, f"{abl} {case} {precision} vs fp64")
    for k in env:
        monkeypatch.delenv(k)
    o = run_gpu(b, precision)
    assert marker not in o["ctx"].path_info()
    compare(b, g, o, FP32_TOL if precision == "fp32" else BF16_EMU_TOL, f"{abl} {case} {precision} vs default engine")


# ------------------------------------------------------------------ pipelined host-buffer steps
def test_train_step_host_async_matches_sync():
    """cavs_train_step_host_async (two steps in flight, sparse root cotangents) gives bit-identical
    dparams to the synchronous host-buffer step on the same batches (same kernels, same order)."""
    bs = [gen.make_batch("tree_lstm", 2, 128, 128, "sst_tree", 6, seed=s) for s in (71, 72, 73)]
    for b in bs[1:]:
        b.params = bs[0].params
    maxV = max(b.V for b in bs)
    ctx = make_ctx(bs[0], "bf16", max_vertices=maxV, max_x=max(b.n_x for b in bs), max_graphs=6)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    ref = []
    for b in bs:
        dp = torch.empty(ctx.P).pin_memory()
        ctx.train_step_host(pin(b.graph_ptr), pin(b.child_ptr), pin(b.child_idx), pin(b.params), pin(b.x),
                            pin(b.x_row), pin(b.gamma), dp)
        ref.append(dp.numpy().copy())
    outs = []
    keep = []
    for rep in range(2):
        for b in bs:
            rows = np.nonzero(np.abs(b.gamma).sum(axis=1))[0].astype(np.int32)
            dp = torch.empty(ctx.P).pin_memory()
            args = (pin(b.graph_ptr), pin(b.child_ptr), pin(b.child_idx), pin(b.params), pin(b.x), pin(b.x_row),
                    pin(b.gamma[rows]), dp)
            keep.append(args)
            ctx.train_step_host_async(*args, gamma_rows=pin(rows))
            outs.append(dp)
    ctx.sync()
    for i, dp in enumerate(outs):
        assert np.array_equal(dp.numpy(), ref[i % 3]), f"async step {i} differs"


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dx_records_pulled_never_or_twice(precision):
    """pull's adjoint with x_row not a bijection: some records pulled by no vertex (their dx
    rows must be 0), some by two vertices (their adjoints ADD); and a bijective batch on the
    same context afterwards (plain stores, no zero fill) still matches the oracle."""
    b = gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 5, seed=81)
    rng = np.random.default_rng(81)
    n_x = b.n_x + 7                                   # 7 records nobody pulls
    x = rng.uniform(-1, 1, size=(n_x, b.d)).astype(np.float32)
    xr = b.x_row.copy()
    has = np.nonzero(xr >= 0)[0]
    xr[has] = rng.permutation(n_x)[:len(has)]
    xr[has[:3]] = xr[has[3:6]]                        # 3 records pulled twice
    b.x, b.x_row = x, xr.astype(np.int32)
    g = run_gpu(b, precision)
    r = run_oracle(b)
    tol = FP32_TOL if precision == "fp32" else BF16_TOL
    compare(b, g, r, tol, f"non-bijective pulls {precision}")
    unused = np.setdiff1d(np.arange(n_x), b.x_row[b.x_row >= 0])
    assert np.all(g["dx"][unused] == 0)
    b2 = gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 5, seed=82)
    g2 = run_gpu(b2, precision, ctx=g["ctx"])
    compare(b2, g2, run_oracle(b2), tol, f"bijective pulls after {precision}")


# ------------------------------------------------------------------ sync-free mode + CUDA graphs
def _dev_step(ctx, b, params_t, x_t, xr_t, g_t, csr, h_out, dp, dx):
    ctx.load_graphs(*csr)
    ctx.schedule(wait=False)
    ctx.forward(params_t, x_t, xr_t, h_out)
    ctx.backward(g_t, dp, dx)


def test_sync_free_step_and_cuda_graph_replay():
    """Sync-free mode: the host never reads the schedule header; the step equals the normal step
    (h_out bit for bit; dparams up to the lazy GEMMs' split order) and a whole step captured in ONE
    CUDA graph replays to the same bits as the uncaptured sync-free step, on two batches."""
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    bs = [gen.make_batch("tree_lstm", 2, 256, 256, "sst_tree", 24, seed=s) for s in (91, 92)]
    for b in bs[1:]:
        b.params = bs[0].params
    maxV = max(b.V for b in bs)
    maxX = max(b.n_x for b in bs)
    ref = [run_gpu(b, "bf16") for b in bs]
    ctx = make_ctx(bs[0], "bf16", max_vertices=maxV, max_x=maxX, max_graphs=24)
    ctx.set_sync_free(True)
    params = t(bs[0].params)
    ins = [(t(b.x), t(b.x_row), t(b.gamma), (t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))) for b in bs]
    outs = [(torch.empty(b.V, b.h, device=dev), torch.empty(ctx.P, device=dev), torch.empty(b.n_x, b.d, device=dev))
            for b in bs]
    for i, b in enumerate(bs):                          # uncaptured sync-free steps
        _dev_step(ctx, b, params, ins[i][0], ins[i][1], ins[i][2], ins[i][3], *outs[i])
        ctx.sync()
        assert np.array_equal(outs[i][0].cpu().numpy(), ref[i]["h_out"])
        compare(b, dict(h_out=outs[i][0].cpu().numpy(), dparams=outs[i][1].cpu().numpy(),
                        dx=outs[i][2].cpu().numpy()), ref[i], 1e-5, f"sync-free vs normal step {i}")
    first = [(o[0].clone(), o[1].clone(), o[2].clone()) for o in outs]
    graphs = []
    side = torch.cuda.Stream(dev)
    for i, b in enumerate(bs):                          # one graph per batch
        g = torch.cuda.CUDAGraph()
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                ctx.set_stream(side)
                _dev_step(ctx, b, params, ins[i][0], ins[i][1], ins[i][2], ins[i][3], *outs[i])
        graphs.append(g)
    ctx.set_stream(torch.cuda.current_stream(dev))
    for rep in range(2):
        for i, g in enumerate(graphs):
            for o in outs[i]:
                o.zero_()
            g.replay()
            torch.cuda.synchronize()
            for a, r in zip(outs[i], first[i]):
                assert torch.equal(a, r), f"graph replay {rep} batch {i} differs"
    ctx.sync()


def test_sync_free_reports_errors_at_sync():
    from paper_1712_04048_b200 import CavsError
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for graphs, code in (([[[1, 2], [2], [0]]], "E_CYCLE"), ([[[], [0, 0], [1, 0]]], "E_UNSUPPORTED")):
        b = gen.batch_from_graphs(graphs, cell="tree_lstm", N=2, h=128, d=128, seed=0, x_at="all", loss_at="all")
        ctx = make_ctx(b, "bf16", max_vertices=16, max_graphs=4, max_x=16)
        ctx.set_sync_free(True)
        ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx))
        ctx.schedule(wait=False)
        ctx.forward(t(b.params), t(b.x), t(b.x_row))
        ctx.backward(t(b.gamma))
        with pytest.raises(CavsError) as e:
            ctx.sync()
        assert e.value.name == code

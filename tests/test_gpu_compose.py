"""NEXT-4: composition through push / pull (Fig. 3, §3.1) -- the fused softmax
head of the language models (reading Z9), the embedding pull, and two vertex functions
wired encoder -> decoder -- against the fp64 oracle wired the same way."""
import numpy as np
import pytest
import torch

import oracle
from gpu_harness import make_ctx, param_blocks, rel
from workloads import gen

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_softmax_xent_matches_the_oracle_head():
    """cavs_softmax_xent against oracle.lm_head with W_out = I, b_out = 0 (logits = H): loss and
    dL/dlogits, rows without a target included; in place and out of place agree bit for bit."""
    from paper_1712_04048_b200.cavs import softmax_xent
    rng = np.random.default_rng(0)
    M, vocab = 37, 1000
    logits = (rng.normal(size=(M, vocab)) * 3).astype(np.float32)
    tgt = rng.integers(0, vocab, size=M).astype(np.int32)
    tgt[[3, 17]] = -1
    L_ref, dl_ref, _, _ = oracle.lm_head(logits, np.eye(vocab), np.zeros(vocab), tgt)
    g = t(logits)
    loss, dl = softmax_xent(g, t(tgt))
    torch.cuda.synchronize()
    assert abs(float(loss.sum()) - L_ref) / abs(L_ref) < 1e-6
    assert rel(dl.cpu().numpy(), dl_ref) < 1e-6
    loss2, dl2 = softmax_xent(g, t(tgt), dlogits=g)
    assert torch.equal(dl2, dl) and torch.equal(loss2, loss)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_lm_train_step(precision, tol):
    """Fixed/Var-LSTM as a language model: embedding pull (x_row = tokens into the embedding table,
    several vertices share a row, their dx ADD up) -> F -> softmax head -> push's adjoint ->
    F backward.  Loss, dparams, d_embedding and the head's gradients against the oracle."""
    from paper_1712_04048_b200 import compose
    lm = gen.make_lm_batch(3, [5, 9, 3], h=64, d=64, vocab=50, seed=4)
    b = lm.batch
    ctx = make_ctx(b, precision, max_x=lm.batch.x.shape[0])
    head = compose.LMHead(t(lm.W_out), t(lm.b_out), tf32=precision == "bf16")
    loss, h_out, dp, demb, dW, db = compose.lm_train_step(
        ctx, t(b.params), t(b.x), t(b.x_row), head, t(lm.targets), graph=(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)))
    torch.cuda.synchronize()
    ho, tape = oracle.forward(b.cell, b.N, b.h, b.d, b.params, b.graph_ptr, b.child_ptr, b.child_idx, b.x_row, b.x)
    L, dH, dW_r, db_r = oracle.lm_head(ho, lm.W_out, lm.b_out, lm.targets)
    dp_r, dx_r = oracle.backward(b.cell, b.N, b.h, b.d, b.params, tape, b.x_row, b.x.shape[0], dH)
    assert abs(float(loss) - L) / abs(L) < tol
    assert rel(h_out.cpu().numpy(), ho) < tol
    for name, sl in param_blocks(b):
        assert rel(dp.cpu().numpy()[sl], dp_r[sl]) < tol, name
    assert rel(demb.cpu().numpy(), dx_r) < tol
    assert rel(dW.cpu().numpy(), dW_r) < tol and rel(db.cpu().numpy(), db_r) < tol


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_encoder_decoder_push_pull(precision, tol):
    """Two vertex functions wired by push / pull: a Tree-LSTM encoder (N = 2) over SST-shaped trees
    pushes its roots' h; decoder chains (LSTM, N = 1, d = h_enc) pull them at their first vertex.
    Forward outputs and both parameter gradients against the oracle wired identically."""
    from paper_1712_04048_b200 import compose
    eb = gen.make_batch("tree_lstm", 2, 64, 64, "sst_tree", 5, seed=7)
    lens = [4, 7, 2, 5, 3]
    db_ = gen.batch_from_graphs([gen.chain(n) for n in lens], cell="tree_lstm", N=1, h=64, d=64, seed=8,
                                x_at="none", loss_at="all")
    roots = compose.roots_of(eb.graph_ptr, eb.child_ptr, eb.child_idx)
    assert len(roots) == eb.K
    dec_xr = -np.ones(db_.V, np.int32)
    dec_xr[db_.graph_ptr[:-1]] = np.arange(eb.K, dtype=np.int32)       # vertex 0 of chain k pulls root k
    enc = make_ctx(eb, precision)
    dec = make_ctx(db_, precision, max_x=eb.K)
    h_enc, h_dec, dpe, dxe, dpd = compose.encoder_decoder_step(
        enc, dec, (t(eb.graph_ptr), t(eb.child_ptr), t(eb.child_idx)), t(eb.params), t(eb.x), t(eb.x_row),
        torch.from_numpy(roots).to(DEV), (t(db_.graph_ptr), t(db_.child_ptr), t(db_.child_idx)), t(db_.params),
        t(dec_xr), t(db_.gamma))
    torch.cuda.synchronize()
    # oracle, same wiring
    he, te = oracle.forward(eb.cell, eb.N, eb.h, eb.d, eb.params, eb.graph_ptr, eb.child_ptr, eb.child_idx,
                            eb.x_row, eb.x)
    xd = he[roots]
    hd, td = oracle.forward(db_.cell, db_.N, db_.h, db_.d, db_.params, db_.graph_ptr, db_.child_ptr, db_.child_idx,
                            dec_xr, xd)
    dpd_r, dxd_r = oracle.backward(db_.cell, db_.N, db_.h, db_.d, db_.params, td, dec_xr, eb.K, db_.gamma)
    ge = np.zeros_like(he)
    ge[roots] = dxd_r
    dpe_r, dxe_r = oracle.backward(eb.cell, eb.N, eb.h, eb.d, eb.params, te, eb.x_row, eb.n_x, ge)
    assert rel(h_enc.cpu().numpy(), he) < tol and rel(h_dec.cpu().numpy(), hd) < tol
    for name, sl in param_blocks(db_):
        assert rel(dpd.cpu().numpy()[sl], dpd_r[sl]) < tol, "decoder " + name
    for name, sl in param_blocks(eb):
        assert rel(dpe.cpu().numpy()[sl], dpe_r[sl]) < tol, "encoder " + name
    assert rel(dxe.cpu().numpy(), dxe_r) < tol

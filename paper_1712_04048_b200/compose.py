"""Composition through push / pull (Fig. 3, §3.1, §4).

A vertex function F only sees the outside world through pull (its input x) and push (its output
h), and their adjoints in the backward pass.  This module wires contexts and the loss
together through exactly those four buffers; every step on the F-over-G path runs in libcavs.so.

* `LMHead` -- the next-word softmax head of the Fixed / Var-LSTM language models, outside
  (F, G) (reading Z9): logits = H W_out^T + b_out and the head's gradient contractions are plain
  GEMMs (cuBLAS through torch.matmul -- library GEMMs), the softmax / cross-entropy / gradient pass
  is the library's fused `cavs_softmax_xent`.
* `lm_train_step` -- embedding pull (x = the embedding table, x_row[v] = token of vertex v; pull's
  adjoint accumulates every vertex's dx into its token's row, cavs.h) -> F forward -> head ->
  push's adjoint dh -> F backward.
* `encoder_decoder_step` -- two vertex functions wired by push / pull: a Tree-LSTM encoder over
  trees pushes its roots' h, which the first vertex of each decoder chain (an LSTM) pulls as x;
  the decoder's dx at those records is the encoder roots' push cotangent.
"""
from __future__ import annotations

import numpy as np

from .cavs import Context, softmax_xent


class LMHead:
    """Softmax head W_out [vocab, h], b_out [vocab] (fp32 device tensors).  `tf32=True` lets the
    head's three GEMMs run on the tensor cores with TF32 inputs (fp32 accumulation and outputs) --
    the precision class of the bf16 mode; the fp32 parity mode keeps exact fp32 GEMMs."""

    def __init__(self, W_out, b_out, tf32=False):
        self.W, self.b, self.tf32 = W_out, b_out, tf32

    def loss_and_grad(self, H, targets):
        """H [V, h] (F's push buffer), targets [V] int32 (-1: no loss).  Returns the summed loss (0-dim
        tensor), dL/dH [V, h] (F's push cotangent), dL/dW_out, dL/db_out."""
        import torch
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = self.tf32
        try:
            logits = torch.addmm(self.b, H, self.W.t())                   # library GEMM
            loss, dlog = softmax_xent(logits, targets, dlogits=logits)     # fused, in place
            dH = dlog @ self.W                                             # library GEMM
            dW = dlog.t() @ H
            db = dlog.sum(0)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        return loss.sum(), dH, dW, db


def lm_train_step(ctx: Context, params, emb, x_row, head: LMHead, targets, graph=None):
    """One language-model training step of F (a chain LSTM, N = 1) over the loaded / given graphs.
    `emb` [vocab, d] is the pull table, `x_row` [V] the token of every vertex.  Returns
    (loss, h_out, dparams, d_emb, dW_out, db_out)."""
    if graph is not None:
        ctx.load_graphs(*graph)
        ctx.schedule(wait=False)
    h_out = ctx.forward(params, emb, x_row)
    loss, dh, dW, db = head.loss_and_grad(h_out, targets)
    dparams, d_emb = ctx.backward(dh.contiguous())
    return loss, h_out, dparams, d_emb, dW, db


def encoder_decoder_step(enc: Context, dec: Context, enc_graph, enc_params, enc_x, enc_x_row, roots,
                         dec_graph, dec_params, dec_x_row, dec_gamma):
    """Tree-LSTM encoder -> LSTM decoder wired by push / pull.  `roots` [K] are the encoder's root
    vertices; decoder vertex v pulls record dec_x_row[v] of the encoder roots' pushed h (-1: none).
    Loss = sum_v <dec_gamma_v, h_dec_v> (external, reading Z9).  Returns (h_enc, h_dec, d_enc_params,
    d_enc_x, d_dec_params)."""
    import torch
    enc.load_graphs(*enc_graph)
    enc.schedule(wait=False)
    h_enc = enc.forward(enc_params, enc_x, enc_x_row)
    dec_x = h_enc.index_select(0, roots).contiguous()     # push (encoder) -> pull records (decoder)
    dec.load_graphs(*dec_graph)
    dec.schedule(wait=False)
    h_dec = dec.forward(dec_params, dec_x, dec_x_row)
    d_dec_params, d_dec_x = dec.backward(dec_gamma)
    dh_enc = torch.zeros_like(h_enc)                      # pull's adjoint -> the encoder's push cotangent
    dh_enc.index_copy_(0, roots, d_dec_x)
    d_enc_params, d_enc_x = enc.backward(dh_enc)
    return h_enc, h_dec, d_enc_params, d_enc_x, d_dec_params


def roots_of(graph_ptr, child_ptr, child_idx) -> np.ndarray:
    """Global ids of the vertices without a parent (host integer work on the CSR)."""
    V = int(graph_ptr[-1])
    has = np.zeros(V, bool)
    for k in range(len(graph_ptr) - 1):
        lo, hi = int(graph_ptr[k]), int(graph_ptr[k + 1])
        for c in child_idx[child_ptr[lo]:child_ptr[hi]]:
            has[lo + int(c)] = True
    return np.nonzero(~has)[0].astype(np.int64)

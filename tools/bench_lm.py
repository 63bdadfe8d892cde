"""Fixed-LSTM language model end to end on one B200 (§5):
embedding pull (x = the 10k x 512 embedding table, x_row = token ids) -> the chain LSTM F (cavs
forward) -> next-word softmax head (cuBLAS GEMMs + the library's fused softmax / cross-entropy)
-> push's adjoint -> cavs backward (dparams, d_embedding).  cfg2 shapes: 64 sequences of 64
tokens, h = d = 512, vocabulary 10,000.  Device time per step by CUDA events (L2 flushed between
steps), reported as tokens/s and the head's share.

    python tools/bench_lm.py [--steps 20] [--warmup 5] [--batch 64] [--seq 64] [--vocab 10000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1712_04048_b200 import Context, compose
from workloads import gen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=64)
    ap.add_argument("--vocab", type=int, default=10000)
    ap.add_argument("--h", type=int, default=512)
    ap.add_argument("--pool", type=int, default=4)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    lms = [gen.make_lm_batch(a.batch, a.seq, h=a.h, d=a.h, vocab=a.vocab, seed=s) for s in range(a.pool)]
    b0 = lms[0].batch
    ctx = Context("tree_lstm", 1, a.h, a.h, precision="bf16", max_graphs=a.batch, max_vertices=b0.V, max_x=a.vocab)
    params, emb = t(b0.params), t(b0.x)
    head = compose.LMHead(t(lms[0].W_out), t(lms[0].b_out), tf32=True)
    pool = [dict(csr=(t(l.batch.graph_ptr), t(l.batch.child_ptr), t(l.batch.child_idx)), xr=t(l.batch.x_row),
                 tg=t(l.targets)) for l in lms]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(i):
        p = pool[i % len(pool)]
        return compose.lm_train_step(ctx, params, emb, p["xr"], head, p["tg"], graph=p["csr"])

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    evs = []
    heads = []
    st = torch.cuda.current_stream(dev)
    for k in range(a.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        loss, *_ = step(a.warmup + k)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = sum(x.elapsed_time(y) for x, y in evs) / a.steps
    # the head alone on the same shapes (GEMMs + fused softmax/xent + gradient GEMMs)
    H = torch.randn(b0.V, a.h, device=dev) * 0.1
    for _ in range(3):
        head.loss_and_grad(H, pool[0]["tg"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        head.loss_and_grad(H, pool[0]["tg"])
    e1.record(st)
    torch.cuda.synchronize()
    head_ms = e0.elapsed_time(e1) / a.steps
    tokens = a.batch * a.seq
    print(json.dumps({"metric": "Fixed-LSTM LM train tokens/s (embedding pull + F fwd/bwd + softmax head)",
                      "value": tokens / (ms / 1000), "unit": "tokens/s", "ms_per_step": ms, "head_ms": head_ms,
                      "config": {"batch": a.batch, "seq_len": a.seq, "vocab": a.vocab, "h": a.h, "precision": "bf16",
                                 "head": "cuBLAS GEMMs (TF32 inputs, fp32 accumulate) + cavs_softmax_xent"},
                      "loss_last": float(loss)}))


if __name__ == "__main__":
    main()

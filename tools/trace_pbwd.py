"""Debug: per-task timeline of the K-split backward kernel (persist_bwd.cu, CAVS_TRACE=1).

Records: 7000 [cta, i | M << 16, task start, MMA done, partials sent, partials received, epilogue end,
barrier out]; 7100 MMA warp [cta, i, loop start, last commit, nt]; 7200 producer [cta, i, first issue]."""
import os, sys
os.environ["CAVS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1712_04048_b200 import Context
from workloads import gen
b = gen.make_config_batch(sys.argv[1] if len(sys.argv) > 1 else "cfg4", seed=0)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
ctx = Context(b.cell, b.N, b.h, b.d, precision="bf16", max_graphs=b.K, max_vertices=b.V, max_x=b.n_x)
print(ctx.path_info())
ws = ctx.workspace[ctx._ws_off + ctx._ws_bytes - (4 << 20): ctx._ws_off + ctx._ws_bytes]
for it in range(5):
    torch.cuda.synchronize()
    ws.zero_()
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)); ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row)); ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
tail = ws.view(torch.int64).cpu().numpy()
n = min(int(tail[0]), (len(tail) - 16) // 8)
rec = tail[8:8 + 8 * n].reshape(n, 8)
R = rec[rec[:, 0] == 7000]
B = rec[rec[:, 0] == 7001]
bo = {(int(c), int(i)): int(t) for c, i, t in zip(B[:, 1], B[:, 2], B[:, 3])}
R = np.concatenate([R, np.array([[bo.get((int(r[1]), int(r[2]) & 0xFFFF), 0)] for r in R])], axis=1)
Mm = rec[rec[:, 0] == 7100]
P = rec[rec[:, 0] == 7200]
it = R[:, 2] & 0xFFFF
M = R[:, 2] >> 16
print("per task, per-CTA durations in us (mean / max over CTAs): M | start->producer issue | MMA loop | "
      "start->done | done->sent | sent->recv | recv->epi end | epi end->barrier out | barrier out->next start")
cta = R[:, 1]
nxt = {}
for c in set(cta.tolist()):
    rows = R[cta == c]
    rows = rows[np.argsort(rows[:, 2] & 0xFFFF)]
    for a, b2 in zip(rows[:-1], rows[1:]):
        nxt[(c, int(a[2]) & 0xFFFF)] = int(b2[3])
pis = {(int(c), int(i)): int(t) for c, i, t in zip(P[:, 1], P[:, 2], P[:, 3])}
mms = {(int(c), int(i)): (int(b2) - int(a)) for c, i, a, b2 in zip(Mm[:, 1], Mm[:, 2], Mm[:, 3], Mm[:, 4])}
for i in sorted(set(it.tolist())):
    r = R[it == i]
    cols = []
    cols.append([(pis.get((int(x[1]), i), x[3]) - x[3]) / 1e3 for x in r])
    cols.append([mms.get((int(x[1]), i), 0) / 1e3 for x in r])
    for a, b2 in ((3, 4), (4, 5), (5, 6), (6, 7), (7, 8)):
        cols.append([(x[b2] - x[a]) / 1e3 for x in r])
    cols.append([(nxt[(int(x[1]), i)] - x[8]) / 1e3 for x in r if (int(x[1]), i) in nxt])
    txt = " | ".join(f"{np.mean(c):5.2f} {np.max(c):5.2f}" if len(c) else "  -  " for c in cols)
    print(f"i={i:3d} M={int(M[it == i].max()):5d} n={len(r):3d} | {txt}")

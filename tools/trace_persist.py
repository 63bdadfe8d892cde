"""Debug: per-task timeline of the persistent level kernels (CAVS_TRACE=1).

Records (persist.cu): epilogue 2000+E [cta, i, level_start, first_done, epi_end, barrier_end, M_t];
producer 3000+E [cta, i, gate_wait_start, gate_pass]."""
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
for it in range(10):
    torch.cuda.synchronize()
    ws.zero_()
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)); ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row)); ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
tail = ws.view(torch.int64).cpu().numpy()
n = min(int(tail[0]), (len(tail) - 16) // 8)
rec = tail[8:8 + 8 * n].reshape(n, 8)
print("records", n)
# epilogue records: word 2 = i | M_t << 16, word 7 = staging-barrier time of the first tile
ep = (rec[:, 0] >= 2000) & (rec[:, 0] < 3000)
st3 = np.where(ep, rec[:, 7], 0)
rec[ep, 7] = rec[ep, 2] >> 16
rec[ep, 2] = rec[ep, 2] & 0xFFFF
for kind in sorted(set(int(k) for k in rec[:, 0] if 2000 <= k < 3000)):
    E = kind - 2000
    R = rec[rec[:, 0] == kind]
    P = rec[rec[:, 0] == 3000 + E]
    print(f"== epilogue kind {kind}: per task i: M_t | start->first done (max over CTAs) | epi end | barrier in->out | "
          f"level span (first start -> last barrier out) | producer gate lag")
    prev_end = None
    for i in sorted(set(R[:, 2])):
        r = R[R[:, 2] == i]
        p = P[P[:, 2] == i + 1] if len(P) else P
        st = r[:, 3].min()
        done = r[:, 4][r[:, 4] > 0]
        fd = (done.max() - st) / 1e3 if len(done) else float("nan")
        ee = (r[:, 5].max() - st) / 1e3
        bi = (r[:, 6].max() - r[:, 5].max()) / 1e3
        span = (r[:, 6].max() - st) / 1e3
        lag = ((p[:, 4] - r[:, 6].max()).max() / 1e3) if len(p) else float("nan")
        gap = (st - prev_end) / 1e3 if prev_end is not None else 0.0
        prev_end = r[:, 6].max()
        s3 = st3[(rec[:, 0] == kind) & (rec[:, 2] == i)]
        s3 = s3[s3 > 0]
        stg = (s3.max() - st) / 1e3 if len(s3) else float("nan")
        print(f"  i={i:3d} M={int(r[0, 7]):5d} | done {fd:7.2f} | epi_end {ee:7.2f} | barrier {bi:6.2f} | "
              f"span {span:7.2f} | gap {gap:6.2f} | gate lag {lag:6.2f} | staged {stg:7.2f}")
# MMA warp (4000+E): [cta, i, first_full, first_tile_committed, -, nt]; producer (5000+E): [cta, i, first_issue]
for kind in sorted(set(int(k) for k in rec[:, 0] if 4000 <= k < 5000)):
    E = kind - 4000
    M_ = rec[rec[:, 0] == kind]
    P5 = rec[rec[:, 0] == 5000 + E]
    print(f"== MMA kind {kind}: per task: nt | producer first issue -> first full (max, mean) | first full -> tile committed (max, mean) | first full -> last box full (max, mean) | ctas")
    for i in sorted(set(M_[:, 2])):
        m = M_[M_[:, 2] == i]
        p = P5[P5[:, 2] == i]
        iss = {int(c): int(t) for c, t in zip(p[:, 1], p[:, 3])}
        lat = np.array([(int(r[3]) - iss[int(r[1])]) / 1e3 for r in m if int(r[1]) in iss])
        mm = (m[:, 4] - m[:, 3]) / 1e3
        lb = (m[:, 5] - m[:, 3]) / 1e3
        ghz = np.where(m[:, 4] > m[:, 3], m[:, 7] / np.maximum(1, m[:, 4] - m[:, 3]), 0)
        print(f"  i={i:3d} nt={int(m[0, 6]):3d} | {lat.max():6.2f} {lat.mean():6.2f} | {mm.max():6.2f} {mm.mean():6.2f} | "
              f"{lb.max():6.2f} {lb.mean():6.2f} | {len(m)} | SM GHz during issue {ghz.mean():.2f}")

# epilogue detail (6000+E): [cta, i, staged, et0 loop end, max thread loop end, after barrier]
for kind in sorted(set(int(k) for k in rec[:, 0] if 6000 <= k < 7000)):
    R6 = rec[rec[:, 0] == kind]
    print(f"== epilogue detail {kind}: staged -> et0 loop end | staged -> slowest thread loop end | -> barrier out (max over CTAs)")
    for i in sorted(set(R6[:, 2])):
        r = R6[R6[:, 2] == i]
        print(f"  i={i:3d} | {((r[:, 4] - r[:, 3]).max()) / 1e3:6.2f} | {((r[:, 5] - r[:, 3]).max()) / 1e3:6.2f} | "
              f"{((r[:, 6] - r[:, 3]).max()) / 1e3:6.2f}")

# per-CTA durations (mean / max over CTAs) of the epilogue records: start->first done | done->epi end |
# epi end->barrier out | barrier out->next start
for kind in sorted(set(int(k) for k in rec[:, 0] if 2000 <= k < 3000)):
    R = rec[rec[:, 0] == kind]
    print(f"== per-CTA durations {kind}: M | start->done | done->epi end | epi end->barrier out | barrier out->next start")
    nxt = {}
    for c in set(R[:, 1].tolist()):
        rows = R[R[:, 1] == c]
        rows = rows[np.argsort(rows[:, 2])]
        for a, b2 in zip(rows[:-1], rows[1:]):
            nxt[(c, int(a[2]))] = int(b2[3])
    for i in sorted(set(R[:, 2].tolist())):
        r = R[R[:, 2] == i]
        cols = [[(x[4] - x[3]) / 1e3 for x in r if x[4] > 0], [(x[5] - x[4]) / 1e3 for x in r if x[4] > 0],
                [(x[6] - x[5]) / 1e3 for x in r], [(nxt[(int(x[1]), i)] - x[6]) / 1e3 for x in r if (int(x[1]), i) in nxt]]
        txt = " | ".join(f"{np.mean(c):5.2f} {np.max(c):5.2f}" if len(c) else "  -  " for c in cols)
        print(f"  i={i:3d} M={int(r[:, 7].max()):5d} n={len(r):3d} | {txt}")

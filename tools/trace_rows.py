"""Debug: per-launch timeline of the row-tiled level kernel (k_rows, CAVS_TRACE=1) at cfg5 (or argv[1]).

Record 7000+E: [cta | lo << 20, t_pdl, t_first_stage, t_acc, t_reduced, t_epi_done, start] (ns after the
CTA's start); printed per launch (task lo): max over CTAs of each mark, and the launch span."""
import os, sys
os.environ["CAVS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1712_04048_b200 import Context
from workloads import gen
b = gen.make_config_batch(sys.argv[1] if len(sys.argv) > 1 else "cfg5", seed=0)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
ctx = Context(b.cell, b.N, b.h, b.d, precision="bf16", max_graphs=b.K, max_vertices=b.V, max_x=b.n_x)
print(ctx.path_info())
ws = ctx.workspace[ctx._ws_off + ctx._ws_bytes - (4 << 20): ctx._ws_off + ctx._ws_bytes]
for it in range(3):
    torch.cuda.synchronize()
    ws.zero_()
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)); ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row)); ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
tail = ws.view(torch.int64).cpu().numpy()
n = min(int(tail[0]), (len(tail) - 16) // 8)
rec = tail[8:8 + 8 * n].reshape(n, 8)
rec = rec[(rec[:, 0] >= 7000) & (rec[:, 0] < 8000)]
lo = rec[:, 1] >> 20
keys = []
for r in rec:
    k = (int(r[0]), int(r[1] >> 20))
    if k not in keys:
        keys.append(k)
starts = {k: rec[(rec[:, 0] == k[0]) & (lo == k[1]), 7] for k in keys}
order = sorted(keys, key=lambda k: starts[k].min())
prev_end = None
print("E   lo      ctas  start_spread  pdl   stage   acc   reduced  epi   | span  gap")
for k in order:
    R = rec[(rec[:, 0] == k[0]) & (lo == k[1])]
    st = R[:, 7]
    end = (st + R[:, 6]).max()
    span = (end - st.min()) / 1e3
    gap = (st.min() - prev_end) / 1e3 if prev_end is not None else 0
    prev_end = end
    m = lambda c: R[:, c].max() / 1e3
    print(f"{k[0]-7000} {k[1]:7d} {len(R):4d} {(st.max()-st.min())/1e3:8.2f}  {m(2):6.2f} {m(3):6.2f} {m(4):6.2f} {m(5):7.2f} {m(6):6.2f} | {span:6.2f} {gap:6.2f}")

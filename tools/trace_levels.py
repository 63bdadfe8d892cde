"""Debug: per-CTA globaltimer trace of the tcgen05 level kernels (CAVS_TRACE=1)."""
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
ws = ctx.workspace[ctx._ws_off + ctx._ws_bytes - (4 << 20): ctx._ws_off + ctx._ws_bytes]
for it in range(int(os.environ.get('TRACE_ITERS', '20'))):
    torch.cuda.synchronize()
    ws.zero_()
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)); ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row)); ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
tail = ws.view(torch.int64).cpu().numpy()
n = tail[0]
rec = tail[8:8 + 8 * n].reshape(n, 8)
rec = rec[rec[:, 0] < 2000]          # k_tc_level records (kind 100 CL + E); k_rows writes 7000 + E
t0 = rec[:, 3].min()
print("records", n)
# per launch (kind, row_lo): CTAs, first start, last end, max per-CTA phase times
import collections
L = collections.OrderedDict()
for r in rec[np.argsort(rec[:, 3])]:
    L.setdefault((int(r[0]), int(r[2]), int(r[7])), []).append(r)
print("kind row_lo rows ctas | launch_us | max setup / done / end per CTA (us) | start since t0 (us)")
for (k, lo, hi), rs in L.items():
    rs = np.array(rs)
    st, en = rs[:, 3].min(), rs[:, 6].max()
    print(k, lo, hi - lo, len(rs), "| %.2f |" % ((en - st) / 1e3),
          "%.2f %.2f %.2f" % (((rs[:, 4] - rs[:, 3]).max()) / 1e3, ((rs[:, 5] - rs[:, 3]).max()) / 1e3,
                              ((rs[:, 6] - rs[:, 3]).max()) / 1e3), "| %.2f" % ((st - t0) / 1e3))

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
for it in range(3):
    ws = ctx.workspace[ctx._ws_off + ctx._ws_bytes - (4 << 20): ctx._ws_off + ctx._ws_bytes]
    torch.cuda.synchronize()
    ws.zero_()
    ctx.load_graphs(t(b.graph_ptr), t(b.child_ptr), t(b.child_idx)); ctx.schedule()
    ctx.forward(t(b.params), t(b.x), t(b.x_row)); ctx.backward(t(b.gamma))
    torch.cuda.synchronize()
tail = ws.view(torch.int64).cpu().numpy()
n = tail[0]
rec = tail[8:8 + 8 * n].reshape(n, 8)
t0 = rec[:, 3].min()
print("records", n)
print("kind block row_lo rows | start setup(us) done(us) end(us) | since first start")
for r in rec[np.argsort(rec[:, 3])][:400]:
    print(r[0], r[1], r[2], r[7] - r[2], "|", "%.2f %.2f %.2f" % ((r[4] - r[3]) / 1e3, (r[5] - r[3]) / 1e3, (r[6] - r[3]) / 1e3),
          "| %.2f" % ((r[3] - t0) / 1e3))

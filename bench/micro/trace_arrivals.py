"""Per-block arrival times at the grid barrier after one FUSED pass (trace build,
BQ_PROX_TRACE=<it>, BQ_PROX_TRACE_THREAD=-3), against each block's z-segment:
which blocks finish last and why."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import _abi  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200.configs import config2_inputs  # noqa: E402
from paper_2307_02043_b200.wpm import DiagPlusLowRank  # noqa: E402

inp = config2_inputs(128)
dev = torch.device("cuda", 0)
v = torch.tensor(inp["v"], dtype=torch.float32, device=dev)
w = DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=torch.float32, device=dev),
                    d=torch.tensor(inp["d"], dtype=torch.float32, device=dev))
prob = D.DualTvProblem(grid=bq.Grid((128, 128, 128)), v=v, w=w, reg=0.05)
ws = D.ProxWorkspace(prob.grid, torch.float32, dev)
ctx = _abi.ctx_for(dev)
from _trace_util import trace_scratch  # noqa: E402
scratch = trace_scratch(ctx, lambda: D.solve_async(prob, ws, eps=1e-300, max_iter=3))
cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
G, K3 = 148, 128
rows = int(os.environ.get("TILE_ROWS", "9"))
tp = -(-128 // rows) * K3
acc = np.zeros(G)
its = [int(a) for a in sys.argv[1:]] or [30, 50, 70, 90]
for it in its:
    os.environ["BQ_PROX_TRACE"] = str(it)
    zero = torch.zeros(4096, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(scratch), ctypes.c_void_p(zero.data_ptr()), ctypes.c_size_t(4096 * 8), 3)
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    torch.cuda.synchronize()
    t = torch.empty(4096, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(scratch), ctypes.c_size_t(4096 * 8), 3)
    torch.cuda.synchronize()
    arr = t.cpu().numpy()[1024:1024 + G].astype(np.float64)
    rel = arr - arr.min()
    acc += rel
    print(f"it {it}: spread {rel.max():.0f} ns, p50 {np.median(rel):.0f}, p90 {np.percentile(rel, 90):.0f}")
acc /= len(its)
b = np.arange(G)
beg, end = b * tp // G, (b + 1) * tp // G
cross = (beg // K3) != ((end - 1) // K3)
z0 = beg % K3
steps = (end - beg) + 1 + (z0 > 0) + cross * 2
order = np.argsort(-acc)
print("slowest blocks (mean ns behind the first): block, ns, planes, steps, crosses, z0, tile")
for i in order[:12]:
    print(f"  {i:3d} {acc[i]:6.0f} {end[i]-beg[i]:3d} {steps[i]:3d} {int(cross[i])} {z0[i]:3d} {beg[i]//K3}")
print("fastest:", [(int(i), int(acc[i])) for i in order[-6:]])
for k in sorted(set(steps)):
    print(f"steps {k}: n={int((steps == k).sum())} mean behind {acc[steps == k].mean():.0f} ns")
sm = np.array([acc[b // K3 == tl].mean() if (beg // K3 == tl).any() else 0 for tl in range(tp // K3)]) if False else None
for tl in range(tp // K3):
    sel = (beg // K3) == tl
    if sel.any():
        print(f"tile {tl}: blocks {int(sel.sum())} mean behind {acc[sel].mean():.0f}")

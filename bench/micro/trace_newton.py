"""Block-0 timeline of the on-chip Newton of one FGP iteration (BQ_PROX_TRACE=<it>, BQ_PROX_TRACE_THREAD=-1)."""
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
zero = torch.zeros(400, dtype=torch.int64, device=dev)
cudart.cudaMemcpy(ctypes.c_void_p(scratch), ctypes.c_void_p(zero.data_ptr()), ctypes.c_size_t(400 * 8), 3)
for _ in range(2):
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
torch.cuda.synchronize()
t = torch.empty(400, dtype=torch.int64, device=dev)
cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(scratch), ctypes.c_size_t(400 * 8), 3)
torch.cuda.synchronize()
a = t.cpu().numpy()
ts = a[240:280]
ts = ts[ts > 0]
print("near entries:", a[300], "stamps:", len(ts))
print("deltas ns:", np.diff(ts).tolist())
if os.environ.get("BQ_PROX_TRACE_THREAD") == "-2":
    prof = a[256:256 + 128]
    ns = prof >> 20
    tot = prof & 0xFFFFF
    sel = ns > 0
    print("per-iteration local Newton ns:", ns[sel].tolist())
    print("near totals:", tot[sel].tolist())

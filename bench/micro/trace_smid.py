"""Per-block arrival at the grid barrier after one FUSED pass against the SM that ran the block
(trace build, BQ_PROX_TRACE_THREAD=-3): is the spread tied to the SM (die) or to the block's work?"""
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
from _trace_util import trace_scratch  # noqa: E402

inp = config2_inputs(128)
dev = torch.device("cuda", 0)
v = torch.tensor(inp["v"], dtype=torch.float32, device=dev)
w = DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=torch.float32, device=dev),
                    d=torch.tensor(inp["d"], dtype=torch.float32, device=dev))
prob = D.DualTvProblem(grid=bq.Grid((128, 128, 128)), v=v, w=w, reg=0.05)
ws = D.ProxWorkspace(prob.grid, torch.float32, dev)
ctx = _abi.ctx_for(dev)
scratch = trace_scratch(ctx, lambda: D.solve_async(prob, ws, eps=1e-300, max_iter=3))
cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
G = 148
acc = np.zeros(G)
its = [30, 40, 50, 60, 70, 80, 90]
for it in its:
    os.environ["BQ_PROX_TRACE"] = str(it)
    zero = torch.zeros(4096, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(scratch), ctypes.c_void_p(zero.data_ptr()), ctypes.c_size_t(4096 * 8), 3)
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    torch.cuda.synchronize()
    t = torch.empty(4096, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(scratch), ctypes.c_size_t(4096 * 8), 3)
    torch.cuda.synchronize()
    a = t.cpu().numpy()
    arr = a[1024:1024 + G].astype(np.float64)
    smid = a[3072:3072 + G]
    acc += arr - arr.min()
acc /= len(its)
print("block smid behind_ns")
for b in range(G):
    print(b, int(smid[b]), int(acc[b]))

"""Dump the block-0 per-step timeline of one FUSED prox pass (BQ_PROX_TRACE=<iteration>)."""
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
for _ in range(3):
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
torch.cuda.synchronize()
rep = D.read_report(ws)
print("phases ms:", [round(x / 1e6, 3) for x in rep.phase_ns], "counts:", list(rep.phase_count))
ctx = _abi.ctx_for(dev)
# scratch lives in the ctx; read it back via a tiny D2H of the raw pointer
import ctypes
buf = np.zeros(240, dtype=np.uint64)
cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
ptr = ctypes.c_void_p()
# ws.scratch is the first pointer after partials/barrier/ctl/ctl_bytes in bq_ctx::ws
from _trace_util import trace_scratch  # noqa: E402
scratch = trace_scratch(ctx, lambda: D.solve_async(prob, ws, eps=1e-300, max_iter=3))
t = torch.empty(240, dtype=torch.int64, device=dev)
cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(scratch), ctypes.c_size_t(240 * 8), 3)
torch.cuda.synchronize()
a = t.cpu().numpy().astype(np.int64).reshape(-1, 4)
a = a[a[:, 0] > 0]
t0 = a[0, 0]
for s, (ta, tb, tc, td) in enumerate(a):
    print(f"step {s:2d}: start {ta - t0:7d} ns  wait {tb - ta:6d}  compute {tc - tb:6d}  sync+release {td - tc:6d}")

"""Block-0 timeline between two FUSED passes (BQ_PROX_TRACE=<it>, BQ_PROX_TRACE_THREAD=-3, trace build):
pass end -> partials written -> barrier complete -> partials reduced -> controller -> on-chip Newton
-> next pass set up -> first stage of the next pass landed."""
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
names = ["pass end", "partials out", "barrier done", "reduced", "controller", "newton", "next set up", "1st stage"]
for it in [int(a) for a in sys.argv[1:]] or [30, 60, 90]:
    os.environ["BQ_PROX_TRACE"] = str(it)
    zero = torch.zeros(400, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(scratch), ctypes.c_void_p(zero.data_ptr()), ctypes.c_size_t(400 * 8), 3)
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    torch.cuda.synchronize()
    t = torch.empty(400, dtype=torch.int64, device=dev)
    cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(scratch), ctypes.c_size_t(400 * 8), 3)
    torch.cuda.synchronize()
    a = t.cpu().numpy()[320:334]
    print("  pass entry -> staged pass entered:", a[11] - a[9], "ns -> march loop:", a[12] - a[11], "ns -> first stage passed:", a[7] - a[12], "ns")
    cyc = t.cpu().numpy()[340:342]
    print("  controller cycles: timeline", cyc[0], "run", cyc[1])
    st = a[:8]
    print("  pass entry after set up:", a[9] - st[6], "ns; pre / prefetched:", a[10] % 100, a[10] // 100)
    print(f"it {it} (ctl it {a[8]}):", "  ".join(f"{names[i]} +{st[i] - st[i - 1]}" for i in range(1, 8) if st[i] and st[i - 1]))

"""Where the end-to-end prox step loses time against the device solve (config 2, 128^3):
device time of one solve, device time of one problem build (validation kernels), host
wall time of a build, and the device gap between consecutive solves in bench.py's
pipelined e2e loop (events recorded around every solve)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200.configs import config2_inputs  # noqa: E402

dev = torch.device("cuda", 0)
n = 128
inp = config2_inputs(n)
grid = bq.Grid((n, n, n))
hs = [torch.from_numpy(inp[k].astype(np.float32)).pin_memory() for k in ("v", "d", "u")]
ds = [h.to(dev) for h in hs]
wsp = D.ProxWorkspace(grid, torch.float32, dev)
iters = inp["iters"]
pp = bench._e2e_problem(grid, inp, *ds)
for _ in range(3):
    D.solve_async(pp, wsp, eps=1e-300, max_iter=iters)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sol, bld, hw = [], [], []
for _ in range(10):
    e0.record(); D.solve_async(pp, wsp, eps=1e-300, max_iter=iters); e1.record(); torch.cuda.synchronize()
    sol.append(e0.elapsed_time(e1))
    t0 = time.perf_counter(); e0.record(); bench._e2e_problem(grid, inp, *ds); e1.record(); torch.cuda.synchronize()
    hw.append(1e3 * (time.perf_counter() - t0)); bld.append(e0.elapsed_time(e1))
print(f"solve device {np.median(sol):.3f} ms; build device {np.median(bld):.3f} ms, host wall {np.median(hw):.3f} ms")
# device gaps in the pipelined loop: wrap solve_async to record events around each solve
evs = []
orig = D.solve_async


def timed(*a, **k):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r = orig(*a, **k); e.record(); evs.append((s, e))
    return r


D.solve_async = timed


class A:
    steps, warmup = 20, 3


ms = bench.e2e_pipelined_ms(A, dev, grid, inp, wsp, *hs, iters)
torch.cuda.synchronize()
tl = evs[-A.steps:]
gaps = [tl[i][1].elapsed_time(tl[i + 1][0]) for i in range(len(tl) - 1)]
durs = [s.elapsed_time(e) for s, e in tl]
print(f"pipelined e2e {ms:.3f} ms/step; solve events {np.median(durs):.3f} ms; gap end(i)->start(i+1) "
      f"median {np.median(gaps):.3f} ms, max {np.max(gaps):.3f} ms")

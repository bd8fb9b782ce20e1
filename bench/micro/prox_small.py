"""Prox solve time and device phases at small grids (config-1 scale, latency-bound)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2307_02043_b200 as bq
from paper_2307_02043_b200 import dual_tv_solver as D
from paper_2307_02043_b200.wpm import DiagPlusLowRank, BoxSet

for n, r, dt in [(32, 1, torch.float64), (32, 4, torch.float64), (64, 4, torch.float64), (32, 1, torch.float32)]:
    N = n ** 3
    rng = np.random.default_rng(0)
    v = torch.tensor(rng.standard_normal(N) * 0.02 + 0.03, dtype=dt, device="cuda")
    U = torch.tensor(rng.standard_normal((N, r)) / np.sqrt(N), dtype=dt, device="cuda")
    w = DiagPlusLowRank(1.25, U)
    prob = D.DualTvProblem(grid=bq.Grid((n, n, n)), v=v, w=w, reg=1e-3, box=BoxSet(0.0, 0.1))
    ws = D.ProxWorkspace(prob.grid, dt, v.device)
    for i in range(3):
        D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(5):
        D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    rep = D.read_report(ws)
    print(f"n={n} r={r} {dt}: {ms:.3f} ms / 100 it ({ms * 10:.1f} us/it); phases ms", [round(x / 1e6, 3) for x in rep.phase_ns],
          "visits", list(rep.phase_count), "newton", rep.newton_iterations)

import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2307_02043_b200 as bq
from paper_2307_02043_b200 import dual_tv_solver as D
from paper_2307_02043_b200.wpm import DiagPlusLowRank, BoxSet
from paper_2307_02043_b200.configs import config2_inputs
for n, r in [(128, 1), (128, 4), (256, 1), (256, 4)]:
    N = n ** 3
    rng = np.random.default_rng(0)
    v = torch.tensor(rng.standard_normal(N) + 0.5, dtype=torch.float32, device="cuda")
    U = torch.tensor(rng.standard_normal((N, r)) / np.sqrt(N), dtype=torch.float32, device="cuda")
    w = DiagPlusLowRank(1.25, U)
    prob = D.DualTvProblem(grid=bq.Grid((n, n, n)), v=v, w=w, reg=0.05, box=BoxSet(0.0, np.inf))
    ws = D.ProxWorkspace(prob.grid, torch.float32, v.device)
    for i in range(2):
        D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(3):
        D.solve_async(prob, ws, eps=1e-300, max_iter=100)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    rep = D.read_report(ws)
    bpv = 4 * (13 + r)
    print(f"n={n} r={r} scalar tau: {ms:.2f} ms, {bpv} B/voxel-iter -> {bpv*N*100/ms/1e6:.0f} GB/s ({bpv*N*100/ms/1e6/6546.6:.2f} of peak); phases", [round(x/1e6,2) for x in rep.phase_ns])

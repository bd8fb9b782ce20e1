"""One prox shape, scalar-tau metric of rank r on an n^3 grid: python bench/micro/prox_one.py n r [solves]"""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2307_02043_b200 as bq
from paper_2307_02043_b200 import dual_tv_solver as D
from paper_2307_02043_b200.wpm import DiagPlusLowRank, BoxSet
n, r = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
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
for i in range(reps):
    D.solve_async(prob, ws, eps=1e-300, max_iter=100)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
rep = D.read_report(ws)
bpv = 4 * (13 + r)
print(f"n={n} r={r} scalar tau: {ms:.3f} ms, {bpv*N*100/ms/1e6/6549.1:.3f} of peak; phases", [round(x/1e6,3) for x in rep.phase_ns], "newton", rep.newton_iterations)

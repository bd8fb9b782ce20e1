"""Oracle fixtures on the EXACT shapes bench.py measures ("pin parity
on the shapes you bench").

Run in the build container (needs /root/reference for the reference solve):

    python tests/golden/make_bench_fixtures.py [prox] [ls] [config3]

Writes tests/golden/bench_*.npz.  The GPU box never runs the oracle at these
sizes; the -m gpu tests read only these files.

* prox     config 2 exactly: 128^3, W = diag(d) + u u^T (d ~ U[0.5, 2],
           u ~ N(0,1)/sqrt(N)), iso TV 0.05, box [0, inf), 100 FGP iterations,
           fp64 numpy port (oracle/prox.py);  plus the scalar-tau twin
           (d == 1.25) solved by the UNMODIFIED reference
           ``tvqn.dual_tv_solver.solve`` (dual_tv_solver.py:161-250).
* ls       config 4 (n = 128 padded to 256^3, L = 64 on a 40 deg cone, 12
           ellipsoids dn ~ U[0.01, 0.1]) at x = x_gt / 2: the subset gradient
           of views {0, 21} with BiCGSTAB tol 1e-6, and one fixed-K (K = 6)
           BiCGSTAB forward solve of view 5, complex128 oracle
           (oracle/physics.py).
* config3  config-3 law at n = 64 (padded 128^3, the pruned-pass size), L = 8,
           K_s = 2, 3 outer iterations, tol 1e-6: the UNMODIFIED reference
           ``bqnpm_run`` (solvers.py:253-317) driving the oracle LS views.

Vectors at 128^3 are stored as a strided sample (every 17th entry, every 51st
for the dual fields; 17 is prime to every grid stride; float32 where the test
tolerance is 1e-4 or looser) plus whole-vector summaries (norm, sum, and the dot
product with a seeded +/-1 vector), so the fixtures stay small while a test
still compares every entry through the summaries.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_SRC = Path("/root/reference/pkg/src")

STRIDE = 17
PROBE_SEED = 99


def probe(n):
    return np.random.default_rng(PROBE_SEED).integers(0, 2, n).astype(float) * 2.0 - 1.0


def summarize(prefix, v, out, stride=STRIDE, dtype=np.float64):
    v = np.asarray(v, dtype=float).reshape(-1)
    out[prefix + "_sample"] = v[::stride].astype(dtype)
    out[prefix + "_norm"] = np.linalg.norm(v)
    out[prefix + "_sum"] = v.sum()
    out[prefix + "_probe"] = v @ probe(v.size)


def make_prox():
    from oracle import prox as O
    from paper_2307_02043_b200.configs import config2_inputs

    inp = config2_inputs(128)
    n = inp["n"]
    out = {}
    t0 = time.time()
    r = O.fgp_prox((n, n, n), inp["v"], O.Metric(U=inp["u"][:, None], d=inp["d"]), reg=inp["reg"],
                   eps=1e-300, max_iter=100)
    summarize("diag_x", r["x"], out)
    summarize("diag_p", r["p_star"], out, stride=3 * STRIDE)
    out["diag_newton"] = r["newton_iterations"]
    out["diag_beta"] = np.asarray(r["beta_star"])
    print(f"config-2 diag(d) port: {time.time() - t0:.1f} s, newton {r['newton_iterations']}")

    sys.path.insert(0, str(REF_SRC))
    from tvqn import dual_tv_solver as DTS
    from tvqn.tv_ops import Grid
    from tvqn.wpm import BoxSet, DiagPlusLowRank

    t0 = time.time()
    prob = DTS.DualTvProblem(grid=Grid((n, n, n)), v=inp["v"], w=DiagPlusLowRank(inp["tau_twin"], inp["u"][:, None]),
                             reg=inp["reg"], box=BoxSet(0.0, np.inf))
    rep = DTS.solve(prob, eps=1e-300, max_iter=100)
    summarize("twin_x", rep.x, out)
    summarize("twin_p", rep.p_star, out, stride=3 * STRIDE)
    out["twin_newton"] = rep.newton_iterations
    out["twin_iterations"] = rep.iterations
    out["twin_beta"] = np.asarray(rep.beta_star)
    print(f"config-2 twin, reference solve: {time.time() - t0:.1f} s, newton {rep.newton_iterations}")
    np.savez_compressed(OUT / "bench_prox128.npz", **out)


def make_ls():
    from oracle import physics as P
    from paper_2307_02043_b200.configs import ls_phantom

    n, L = 128, 64
    s = P.Setup(n=n, n_views=L, theta_deg=40.0)
    m = P.ScatterModel(s, "ls", tol=1e-6, max_iter=500)
    xgt = ls_phantom(n, 12, 0.01, 0.1, seed=4000)
    x = 0.5 * xgt
    out = {}
    views = [0, 21]
    t0 = time.time()
    ys = []
    for l in views:
        ys.append(m.forward(xgt, l))  # noiseless data at the truth; the residual at x_gt/2 is O(1)
    out["views"] = np.array(views)
    out["y"] = np.array(ys).astype(np.float32)  # the device works in complex64
    ys = [y.astype(np.float32).astype(float) for y in ys]
    m.last_iters.clear()
    g = sum(m.gradient(x, l, y) for l, y in zip(views, ys)) / len(views)
    out["grad_iters"] = np.array(m.last_iters)
    summarize("grad", g, out, dtype=np.float32)
    print(f"config-4 gradient, 2 views: {time.time() - t0:.1f} s, iterations {m.last_iters}")
    # fixed-K BiCGSTAB: K = 6 iterations of the forward solve of view 5 (tol 0: never met)
    t0 = time.time()
    f, _ = m.pot(x)
    uin = P.incident(s, 5).reshape(-1)
    u6, it, res = P.bicgstab(lambda v: v - m.G.dom(f * v), uin, tol=0.0, max_iter=6)
    assert it == 6
    summarize("bicg6_re", u6.real, out, dtype=np.float32)
    summarize("bicg6_im", u6.imag, out, dtype=np.float32)
    out["bicg6_res"] = res
    print(f"config-4 fixed-K BiCGSTAB: {time.time() - t0:.1f} s, residual {res:.3e}")
    np.savez_compressed(OUT / "bench_ls128.npz", **out)


def make_config3():
    sys.path.insert(0, str(REF_SRC))
    from tvqn import forward_models as fm
    from tvqn import solvers
    from tvqn.tv_ops import Grid
    from tvqn.wpm import BoxSet

    from oracle import physics as P
    from paper_2307_02043_b200.configs import complex_noise, ls_phantom
    from make_golden import scaled_adjoint_x0

    n, L = 64, 8
    s = P.Setup(n=n, n_views=L, theta_deg=35.0)
    m = P.ScatterModel(s, "ls", tol=1e-6, max_iter=500)
    xgt = ls_phantom(n, 5, 0.02, 0.08, seed=3000)
    rng = np.random.default_rng(3001)
    ys = []
    for l in range(L):
        y = m.forward(xgt, l)
        ys.append(y + complex_noise(y, 30.0, rng))
    views = [fm.ViewProblem(lambda x, l=l: m.forward(x, l), lambda x, v, l=l: m.jvp(x, l, v),
                            lambda x, z, l=l: m.vjp(x, l, z), ys[l], view_id=l) for l in range(L)]
    grid = Grid((n, n, n))
    box = BoxSet(0.0, 0.1)
    t0 = time.time()
    x0 = scaled_adjoint_x0(views, box, n ** 3)
    print(f"config-3 x0: {time.time() - t0:.1f} s")
    parts = solvers.partition_views(L, 2)
    alphas = solvers.estimate_subset_lipschitz(views, parts, x0, 2, 1.05, 0)
    print(f"config-3 alphas {alphas}: {time.time() - t0:.1f} s")
    cfg = solvers.SolverConfig(subsets=2, tv_weight=1e-3, max_outer=3, box=box, seed=0, alphas=alphas)
    x, tr = solvers.bqnpm_run(views, grid, cfg, x0=x0, ground_truth=xgt)
    f32 = np.float32
    out = {"y": np.array(ys).astype(f32), "x0": x0.astype(f32), "alphas": alphas, "x": x.astype(f32),
           "cost": tr.column("cost"),
           "inner": tr.column("inner_iters"), "snr": tr.column("snr_db")}
    np.savez_compressed(OUT / "bench_config3_64.npz", **out)
    print(f"config-3 n=64 bqnpm: {time.time() - t0:.1f} s, snr {tr.column('snr_db')}")


if __name__ == "__main__":
    sys.path.insert(0, str(OUT))
    which = sys.argv[1:] or ["prox", "ls", "config3"]
    for w in which:
        {"prox": make_prox, "ls": make_ls, "config3": make_config3}[w]()

"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``)
and its independent dense test oracles (``/root/reference/pkg/tests/oracles.py``),
evaluates them on seeded inputs, and writes ``tests/golden/*.npz``.  The
GPU box never sees /root/reference: tests there read only these fixtures.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(REF / "tests"))
    import tvqn  # noqa: F401
    from tvqn import dual_tv_solver, forward_models, hessian_sr1, solvers, tv_ops, wpm
    import oracles

    return tv_ops, wpm, dual_tv_solver, hessian_sr1, solvers, forward_models, oracles


def main(which=None):
    tv_ops, wpm, dts, sr1, solvers, fm, oracles = _import_reference()
    if which:
        for w in which:
            {"config1": make_config1_golden, "config3s": make_config3_small_golden,
             "baselines": make_baselines_golden, "formats": make_formats_golden}[w](tv_ops, wpm, solvers, fm)
        return
    Grid, TvMode = tv_ops.Grid, tv_ops.TvMode
    out = {}

    # ---- stencils and TV value (tv_ops.py:107-167) ------------------------
    rng = np.random.default_rng(101)
    for dims in [(7,), (5, 4), (4, 3, 2), (6, 5, 4)]:
        g = Grid(dims)
        x = rng.standard_normal(g.size)
        p = rng.standard_normal((g.ndim, g.size))
        key = "x".join(map(str, dims))
        out[f"stencil_{key}_x"] = x
        out[f"stencil_{key}_p"] = p
        out[f"stencil_{key}_grad"] = tv_ops.gradient_stack(g, x)
        out[f"stencil_{key}_div"] = tv_ops.dual_divergence(g, p)
        out[f"stencil_{key}_tv_iso"] = np.array(tv_ops.tv_value(g, x, TvMode.ISOTROPIC))
        out[f"stencil_{key}_tv_aniso"] = np.array(tv_ops.tv_value(g, x, TvMode.ANISOTROPIC))
        out[f"stencil_{key}_proj_iso"] = tv_ops.project_dual(2.0 * p, TvMode.ISOTROPIC)
        out[f"stencil_{key}_proj_aniso"] = tv_ops.project_dual(2.0 * p, TvMode.ANISOTROPIC)

    # ---- metric apply / inverse (wpm.py:81-106) ---------------------------
    rng = np.random.default_rng(202)
    for i, (n, r, sign, scale) in enumerate([(64, 0, 1, 1.0), (64, 1, 1, 1.0), (256, 4, 1, 1.0),
                                             (32, 2, -1, 0.08), (100, 8, 1, 2.0)]):
        tau = float(rng.uniform(0.5, 2.0))
        u = scale * rng.standard_normal((n, r)) / (np.sqrt(n) if sign > 0 else 1.0)
        w = wpm.DiagPlusLowRank(tau, u, sign=sign)
        x = rng.standard_normal(n)
        out[f"metric{i}_tau"] = np.array(tau)
        out[f"metric{i}_U"] = u
        out[f"metric{i}_sign"] = np.array(sign)
        out[f"metric{i}_x"] = x
        out[f"metric{i}_Wx"] = wpm.apply_metric(w, x)
        out[f"metric{i}_Winvx"] = wpm.apply_metric_inverse(w, x)

    # ---- wpm_box (wpm.py:234-253) -----------------------------------------
    rng = np.random.default_rng(303)
    cases = [(200, 1, 0.0, np.inf, None), (200, 3, -0.5, 1.5, None), (500, 2, 0.0, np.inf, "warm"),
             (64, 4, 0.0, 0.1, None)]
    for i, (n, r, lo, hi, warm) in enumerate(cases):
        tau = float(rng.uniform(0.5, 2.0))
        u = rng.standard_normal((n, r)) / np.sqrt(n) * 3.0
        w = wpm.DiagPlusLowRank(tau, u)
        x = rng.standard_normal(n)
        beta0 = rng.standard_normal(r) * 0.1 if warm else None
        uo, info = wpm.wpm_box(x, w, wpm.BoxSet(lo, hi), beta0=beta0, full_output=True)
        out[f"wpm{i}_tau"] = np.array(tau)
        out[f"wpm{i}_U"] = u
        out[f"wpm{i}_x"] = x
        out[f"wpm{i}_lo"] = np.array(lo)
        out[f"wpm{i}_hi"] = np.array(hi)
        out[f"wpm{i}_beta0"] = np.zeros(r) if beta0 is None else beta0
        out[f"wpm{i}_has_beta0"] = np.array(beta0 is not None)
        out[f"wpm{i}_u"] = uo
        out[f"wpm{i}_beta"] = info["beta"]
        out[f"wpm{i}_iters"] = np.array(info["iterations"])

    # ---- prox solve (dual_tv_solver.py:161-250) ---------------------------
    rng = np.random.default_rng(404)
    prox_cases = [
        # dims, rank, reg, mode, lo, hi, eps, max_iter, accelerated, tau, warm
        ((8, 8), 1, 0.3, "iso", 0.0, np.inf, 1e-5, 100, True, 1.0, False),
        ((6, 6), 1, 0.3, "aniso", 0.0, np.inf, 1e-5, 100, True, 1.3, False),
        ((8, 8), 2, 0.5, "iso", 0.0, np.inf, 1e-5, 30, True, 0.7, False),
        ((6, 6), 1, 0.4, "iso", 0.0, np.inf, 1e-15, 1, False, 1.0, True),
        ((4, 4, 4), 1, 0.3, "iso", 0.0, np.inf, 1e-5, 100, True, 1.0, False),
        ((16, 16, 16), 1, 0.05, "iso", 0.0, np.inf, 1e-300, 40, True, 1.25, False),
        ((12, 10, 8), 4, 0.02, "iso", 0.0, 0.1, 1e-5, 100, True, 3.0, True),
        ((24, 24, 24), 1, 0.05, "iso", 0.0, np.inf, 1e-300, 100, True, 1.25, False),
        ((10, 9, 7), 0, 0.1, "aniso", -0.2, 0.5, 1e-5, 60, True, 2.0, False),
        ((9, 7), 3, 0.0, "iso", 0.0, np.inf, 1e-5, 100, True, 1.0, True),
        ((33, 17), 1, 0.2, "iso", 0.0, np.inf, 1e-8, 200, True, 0.9, False),
        ((20,), 1, 0.3, "iso", 0.0, np.inf, 1e-6, 100, True, 1.0, False),
    ]
    for i, (dims, r, reg, mode, lo, hi, eps, mi, acc, tau, warm) in enumerate(prox_cases):
        g = Grid(dims)
        v = rng.standard_normal(g.size) * 0.5 + 0.3
        u = rng.standard_normal((g.size, r)) / np.sqrt(g.size)
        w = wpm.DiagPlusLowRank(tau, u) if r else wpm.DiagPlusLowRank.diagonal(tau, g.size)
        p0 = 0.3 * rng.standard_normal((g.ndim, g.size)) if warm else None
        b0 = 0.01 * rng.standard_normal(r) if (warm and r) else None
        prob = dts.DualTvProblem(grid=g, v=v, w=w, reg=reg, mode=mode, box=wpm.BoxSet(lo, hi),
                                 warm_start=p0, beta_warm=b0)
        rep = dts.solve(prob, eps=eps, max_iter=mi, accelerated=acc)
        k = f"prox{i}"
        out[k + "_dims"] = np.array(dims)
        out[k + "_rank"] = np.array(r)
        out[k + "_reg"] = np.array(reg)
        out[k + "_iso"] = np.array(mode == "iso")
        out[k + "_lo"] = np.array(lo)
        out[k + "_hi"] = np.array(hi)
        out[k + "_eps"] = np.array(eps)
        out[k + "_max_iter"] = np.array(mi)
        out[k + "_acc"] = np.array(acc)
        out[k + "_tau"] = np.array(tau)
        out[k + "_v"] = v
        out[k + "_U"] = u
        out[k + "_has_warm"] = np.array(bool(warm))
        out[k + "_p0"] = p0 if p0 is not None else np.zeros((g.ndim, g.size))
        out[k + "_b0"] = b0 if b0 is not None else np.zeros(r)
        out[k + "_x"] = rep.x
        out[k + "_p_star"] = np.asarray(rep.p_star)
        out[k + "_iterations"] = np.array(rep.iterations)
        out[k + "_rel"] = np.array(rep.rel_change)
        out[k + "_converged"] = np.array(rep.converged)
        out[k + "_newton"] = np.array(rep.newton_iterations)
        out[k + "_beta"] = np.asarray(rep.beta_star if rep.beta_star is not None else np.zeros(0))
    out["prox_count"] = np.array(len(prox_cases))

    # ---- diag(d) extension pinned by the reference's Condat-Vu dense oracle
    rng = np.random.default_rng(505)
    for i, (dims, iso) in enumerate([((8, 8), True), ((6, 6), False), ((4, 4, 3), True)]):
        n = int(np.prod(dims))
        d = rng.uniform(0.5, 2.0, n)
        u = rng.standard_normal((n, 1)) / np.sqrt(n)
        v = rng.standard_normal(n)
        reg = 0.3
        wd = np.diag(d) + u @ u.T
        xref = oracles.condat_vu_tv(dims, wd, v, reg, 0.0, np.inf, iters=40000, isotropic=iso)
        out[f"diag{i}_dims"] = np.array(dims)
        out[f"diag{i}_iso"] = np.array(iso)
        out[f"diag{i}_d"] = d
        out[f"diag{i}_U"] = u
        out[f"diag{i}_v"] = v
        out[f"diag{i}_reg"] = np.array(reg)
        out[f"diag{i}_x_cv"] = xref
        out[f"diag{i}_obj_cv"] = np.array(oracles.tv_objective(dims, wd, v, reg, xref, isotropic=iso))

    # ---- SR1 (hessian_sr1.py:52-101) ---------------------------------------
    rng = np.random.default_rng(606)
    s_list, m_list, tau_l, u_l, has_l = [], [], [], [], []
    for trial in range(40):
        n = 50
        s = rng.standard_normal(n)
        if trial % 4 == 0:
            m = -s  # negative curvature -> fallback
        elif trial % 4 == 1:
            m = 2.0 * s + 1e-3 * rng.standard_normal(n)
        elif trial % 4 == 2:
            a = rng.standard_normal((n, n))
            m = (a @ a.T / n + 0.5 * np.eye(n)) @ s
        else:
            m = rng.standard_normal(n)
        est = sr1.estimate_sr1(s, m, gamma=0.8, alpha_fallback=1.7)
        s_list.append(s)
        m_list.append(m)
        tau_l.append(est.tau)
        has_l.append(est.u is not None)
        u_l.append(est.u if est.u is not None else np.zeros(n))
    out["sr1_s"] = np.array(s_list)
    out["sr1_m"] = np.array(m_list)
    out["sr1_tau"] = np.array(tau_l)
    out["sr1_u"] = np.array(u_l)
    out["sr1_has_u"] = np.array(has_l)

    # ---- aggregate_metric + compute_v_k (solvers.py:67-89) ----------------
    rng = np.random.default_rng(707)
    n = 300
    slots = []
    for t in range(4):
        x = rng.standard_normal(n)
        g = rng.standard_normal(n)
        u = rng.standard_normal(n) / np.sqrt(n) if t != 2 else None
        tau = float(rng.uniform(0.5, 2.0))
        slots.append(solvers.SubsetSlot(x=x, grad=g, hess=sr1.Sr1Estimate(tau=tau, u=u)))
        out[f"vk_x{t}"] = x
        out[f"vk_g{t}"] = g
        out[f"vk_tau{t}"] = np.array(tau)
        out[f"vk_u{t}"] = u if u is not None else np.zeros(n)
        out[f"vk_has_u{t}"] = np.array(u is not None)
    w = solvers.aggregate_metric(slots)
    out["vk_v"] = solvers.compute_v_k(slots, w, 0.7)
    out["vk_tau_w"] = np.array(w.tau)
    out["vk_U_w"] = w.U

    # ---- schedule (solvers.py:29-55) ---------------------------------------
    out["kappa_table"] = np.array([[solvers.kappa(k, t, 4) for t in range(1, 5)] for k in range(1, 13)])
    out["partition_equi_30_4"] = np.concatenate(solvers.partition_views(30, 4))
    out["partition_contig_30_4"] = np.concatenate(solvers.partition_views(30, 4, "contiguous"))

    # ---- DCT stand-in views + BQNPM (forward_models.py, solvers.py) ------
    for tag, strength, snr, dims in [("lin", 0.0, 30.0, (10, 9, 8)), ("nl", 0.1, 30.0, (12, 8, 6))]:
        g = Grid(dims)
        L = 8
        views = (fm.make_linear_views(g, L, mask_fraction=0.5, seed=3, noise_snr_db=snr) if strength == 0.0 else
                 fm.make_nonlinear_views(g, L, strength=strength, mask_fraction=0.5, seed=3, noise_snr_db=snr))
        rng = np.random.default_rng(909)
        x = 1.333 + 0.01 * rng.standard_normal(g.size)
        out[f"views_{tag}_dims"] = np.array(dims)
        out[f"views_{tag}_y"] = np.array([v.y for v in views])
        out[f"views_{tag}_x"] = x
        out[f"views_{tag}_grad_sub"] = fm.subset_gradient(views, [1, 4, 6], x)
        out[f"views_{tag}_values"] = np.array([v.value(x) for v in views])
        out[f"views_{tag}_fwd0"] = views[0].forward(x)
        out[f"views_{tag}_phantom"] = fm.make_phantom(g, seed=3).values
        cfg = solvers.SolverConfig(subsets=4, tv_weight=2e-3, max_outer=10, box=wpm.BoxSet(1.3, 1.4), seed=0)
        xr, tr = solvers.bqnpm_run(views, g, cfg)
        out[f"bqnpm_{tag}_x"] = xr
        out[f"bqnpm_{tag}_cost"] = tr.column("cost")
        out[f"bqnpm_{tag}_inner"] = tr.column("inner_iters")
        parts = solvers.partition_views(L, 4)
        x0 = solvers.default_initializer(views, g, wpm.BoxSet(1.3, 1.4))
        out[f"bqnpm_{tag}_x0"] = x0
        out[f"bqnpm_{tag}_alphas"] = solvers.estimate_subset_lipschitz(views, parts, x0, 30, 1.05, 0)

    np.savez_compressed(OUT / "reference_golden.npz", **out)
    print(f"wrote {OUT / 'reference_golden.npz'} ({len(out)} arrays)")
    make_config1_golden(tv_ops, wpm, solvers, fm)
    make_config3_small_golden(tv_ops, wpm, solvers, fm)
    make_baselines_golden(tv_ops, wpm, solvers, fm)


def make_formats_golden(tv_ops, wpm, solvers, fm):
    """Files written by the REFERENCE harness itself (experiment_cli.py:35-137):
    a TVQNVOL1 volume and a "tvqn-trace v1" CSV, for byte-level format parity."""
    from tvqn import experiment_cli as E

    rng = np.random.default_rng(12)
    x = rng.standard_normal((5, 4, 3))
    E.dump_volume(x, OUT / "ref_volume_5x4x3.tvqnvol")
    tr = solvers.IterationTrace(solver="bqnpm")
    for k in range(4):
        tr.rows.append(solvers.TraceRow(iteration=k, cost=float(1 / (k + 1) + 1e-13 * k), snr_db=float(3.25 * k + 1 / 3),
                                        elapsed_s=0.125 * k, inner_iters=7 * k, grad_evals=k, full_grad_evals=0))
    E.write_trace(tr, OUT / "ref_trace_v1.csv")
    np.savez(OUT / "ref_formats.npz", volume=x)


def make_baselines_golden(tv_ops, wpm, solvers, fm):
    """The REFERENCE aspm_run (momentum on / off) and sqnpm_run (solvers.py:320-422)
    on the same DCT stand-in views as the bqnpm goldens."""
    out = {}
    for tag, strength, snr, dims in [("lin", 0.0, 30.0, (10, 9, 8)), ("nl", 0.1, 30.0, (12, 8, 6))]:
        g = tv_ops.Grid(dims)
        L = 8
        views = (fm.make_linear_views(g, L, mask_fraction=0.5, seed=3, noise_snr_db=snr) if strength == 0.0 else
                 fm.make_nonlinear_views(g, L, strength=strength, mask_fraction=0.5, seed=3, noise_snr_db=snr))
        for name, runner, kw in [("aspm", solvers.aspm_run, dict(max_outer=10)),
                                 ("aspm_plain", solvers.aspm_run, dict(max_outer=10, momentum=False)),
                                 ("sqnpm", solvers.sqnpm_run, dict(max_outer=13))]:
            cfg = solvers.SolverConfig(subsets=4, tv_weight=2e-3, box=wpm.BoxSet(1.3, 1.4), seed=0, **kw)
            xr, tr = runner(views, g, cfg)
            out[f"{name}_{tag}_x"] = xr
            out[f"{name}_{tag}_cost"] = tr.column("cost")
            out[f"{name}_{tag}_inner"] = tr.column("inner_iters")
            out[f"{name}_{tag}_grad_evals"] = tr.column("grad_evals")
            out[f"{name}_{tag}_full_grad_evals"] = tr.column("full_grad_evals")
    np.savez_compressed(OUT / "baselines_golden.npz", **out)
    print(f"wrote {OUT / 'baselines_golden.npz'} ({len(out)} arrays)")


def scaled_adjoint_x0(views, box, N):
    """Numpy statement of ``solvers.scaled_adjoint_initializer`` (the device
    initial guess for the physics views): g0 = mean_rho J^T y_rho at x = 0,
    alpha = ||g0||^2 / <g0, mean_rho J^T J g0>, x0 = clamp(alpha g0)."""
    zero = np.zeros(N)
    L = len(views)
    g0 = sum(v.adjoint_vec(zero, v.y) for v in views) / L
    hg = sum(v.adjoint_vec(zero, v.jacobian_vec(zero, g0)) for v in views) / L
    den = float(g0 @ hg)
    alpha = float(g0 @ g0) / den if den > 0 else 0.0
    return np.clip(alpha * g0, box.lower, box.upper)


def make_config1_golden(tv_ops, wpm, solvers, fm):
    """Config 1 end to end: the REFERENCE bqnpm_run driving the builder's CPU
    first-Born oracle (oracle/physics.py, complex128) through the reference's
    own ViewProblem plugin type (forward_models.py:25-83)."""
    import time

    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    from oracle import physics as P
    from paper_2307_02043_b200.configs import born_spheres_phantom, complex_noise

    n, L = 32, 16
    s = P.Setup(n=n, n_views=L, theta_deg=35.0)
    m = P.ScatterModel(s, "born")
    xgt = born_spheres_phantom(n, seed=1000)
    rng = np.random.default_rng(1001)
    ys = []
    for l in range(L):
        y = m.forward(xgt, l)
        ys.append(y + complex_noise(y, 30.0, rng))
    views = [fm.ViewProblem(lambda x, l=l: m.forward(x, l), lambda x, v, l=l: m.jvp(x, l, v),
                            lambda x, z, l=l: m.vjp(x, l, z), ys[l], view_id=l) for l in range(L)]
    grid = tv_ops.Grid((n, n, n))
    box = wpm.BoxSet(0.0, 0.1)
    t0 = time.time()
    x0 = scaled_adjoint_x0(views, box, n ** 3)
    parts = solvers.partition_views(L, 4)
    alphas = solvers.estimate_subset_lipschitz(views, parts, x0, 30, 1.05, 0)
    cfg = solvers.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=20, box=box, seed=0, alphas=alphas)
    x, tr = solvers.bqnpm_run(views, grid, cfg, x0=x0, ground_truth=xgt)
    out = {"c1_y": np.array(ys), "c1_xgt": xgt, "c1_x0": x0, "c1_alphas": alphas, "c1_x": x,
           "c1_cost": tr.column("cost"), "c1_inner": tr.column("inner_iters"), "c1_snr": tr.column("snr_db"),
           "c1_x0_reference_initializer": solvers.default_initializer(views, grid, box)}
    np.savez_compressed(OUT / "config1_golden.npz", **out)
    print(f"wrote config1_golden.npz in {time.time() - t0:.1f} s; final SNR {tr.column('snr_db')[-1]:.2f} dB")




def make_config3_small_golden(tv_ops, wpm, solvers, fm):
    """Config 3 law at reduced size (LS, n=20 padded to 40^3, L=8, K_s=4, 4 outer
    iterations, 5 ellipsoids dn~U[0.02,0.08], 30 dB): the REFERENCE bqnpm_run
    driving the CPU LS oracle with converged BiCGSTAB (tol 1e-12)."""
    import time

    sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
    from oracle import physics as P
    from paper_2307_02043_b200.configs import complex_noise, ls_phantom

    n, L = 20, 8
    s = P.Setup(n=n, n_views=L, theta_deg=35.0)
    m = P.ScatterModel(s, "ls", tol=1e-12, max_iter=1000)
    xgt = ls_phantom(n, 5, 0.02, 0.08, seed=3000)
    rng = np.random.default_rng(3001)
    ys = []
    for l in range(L):
        y = m.forward(xgt, l)
        ys.append(y + complex_noise(y, 30.0, rng))
    views = [fm.ViewProblem(lambda x, l=l: m.forward(x, l), lambda x, v, l=l: m.jvp(x, l, v),
                            lambda x, z, l=l: m.vjp(x, l, z), ys[l], view_id=l) for l in range(L)]
    grid = tv_ops.Grid((n, n, n))
    box = wpm.BoxSet(0.0, 0.1)
    t0 = time.time()
    x0 = solvers.default_initializer(views, grid, box)
    parts = solvers.partition_views(L, 4)
    alphas = solvers.estimate_subset_lipschitz(views, parts, x0, 10, 1.05, 0)
    cfg = solvers.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=4, box=box, seed=0, alphas=alphas)
    x, tr = solvers.bqnpm_run(views, grid, cfg, x0=x0, ground_truth=xgt)
    out = {"c3_y": np.array(ys), "c3_xgt": xgt, "c3_x0": x0, "c3_alphas": alphas, "c3_x": x,
           "c3_cost": tr.column("cost"), "c3_inner": tr.column("inner_iters")}
    np.savez_compressed(OUT / "config3s_golden.npz", **out)
    print(f"wrote config3s_golden.npz in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main(sys.argv[1:])

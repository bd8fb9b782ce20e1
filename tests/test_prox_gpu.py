"""Parity of the device prox / WPM / metric path (through the C ABI) against the
reference golden vectors and the CPU oracle.  Tolerances (north star):
fp64 <= 1e-10 relative L2, fp32 <= 1e-4."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import prox as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200 import wpm as W  # noqa: E402

F64_TOL = 1e-10
F32_TOL = 1e-4


def _prox_problem(golden, i, dtype=None):
    k = f"prox{i}"
    dims = tuple(int(v) for v in golden[k + "_dims"])
    r = int(golden[k + "_rank"])
    n = int(np.prod(dims))
    tau = float(golden[k + "_tau"])
    if dtype is None:
        w = W.DiagPlusLowRank(tau, golden[k + "_U"]) if r else W.DiagPlusLowRank.diagonal(tau, n)
        v = golden[k + "_v"]
    else:
        u = torch.tensor(golden[k + "_U"], dtype=dtype, device="cuda")
        w = W.DiagPlusLowRank(tau, u) if r else W.DiagPlusLowRank.diagonal(tau, n, dtype=dtype)
        v = torch.tensor(golden[k + "_v"], dtype=dtype, device="cuda")
    warm = bool(golden[k + "_has_warm"])
    prob = D.DualTvProblem(
        grid=bq.Grid(dims), v=v, w=w, reg=float(golden[k + "_reg"]),
        mode="iso" if bool(golden[k + "_iso"]) else "aniso",
        box=W.BoxSet(float(golden[k + "_lo"]), float(golden[k + "_hi"])),
        warm_start=golden[k + "_p0"] if warm else None,
        beta_warm=golden[k + "_b0"] if (warm and r) else None,
    )
    kw = dict(eps=float(golden[k + "_eps"]), max_iter=int(golden[k + "_max_iter"]),
              accelerated=bool(golden[k + "_acc"]))
    return prob, kw


@pytest.mark.parametrize("i", range(12))
def test_prox_f64_matches_reference_golden(golden, i):
    prob, kw = _prox_problem(golden, i)
    rep = D.solve(prob, **kw)
    k = f"prox{i}"
    assert isinstance(rep.x, np.ndarray)
    assert rel_l2(rep.x, golden[k + "_x"]) <= F64_TOL
    assert rel_l2(rep.p_star, golden[k + "_p_star"]) <= F64_TOL
    assert rep.iterations == int(golden[k + "_iterations"])
    assert rep.converged == bool(golden[k + "_converged"])
    assert rep.newton_iterations == int(golden[k + "_newton"])
    if int(golden[k + "_rank"]):
        bref = golden[k + "_beta"]
        assert np.max(np.abs(rep.beta_star - bref)) <= 1e-8 * max(1.0, float(np.max(np.abs(bref))))
    assert np.all(rep.x >= float(golden[k + "_lo"])) and np.all(rep.x <= float(golden[k + "_hi"]))


@pytest.mark.parametrize("i", [0, 4, 5, 7, 10])
def test_prox_f32_close_to_reference(golden, i):
    prob, kw = _prox_problem(golden, i, dtype=torch.float32)
    # fixed iteration count so fp32 roundoff cannot move the stopping decision
    kw["eps"] = 1e-300
    rep = D.solve(prob, **kw)
    ref = O.fgp_prox(prob.grid.dims, golden[f"prox{i}_v"],
                     O.Metric(tau=prob.w.tau, U=golden[f"prox{i}_U"] if prob.w.rank else None, n=prob.grid.size),
                     reg=prob.reg, lo=float(golden[f"prox{i}_lo"]), hi=float(golden[f"prox{i}_hi"]),
                     isotropic=prob.mode.value == "isotropic", eps=1e-300, max_iter=kw["max_iter"],
                     accelerated=kw["accelerated"])
    assert rep.x.dtype == torch.float32
    assert rel_l2(rep.x.cpu().numpy(), ref["x"]) <= F32_TOL
    assert rel_l2(rep.p_star.cpu().numpy(), ref["p_star"]) <= F32_TOL


def _diag_problem(seed, dims, r=1, reg=0.05, iso=True, lo=0.0, hi=np.inf):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    d = rng.uniform(0.5, 2.0, n)
    u = rng.standard_normal((n, r)) / np.sqrt(n)
    v = rng.standard_normal(n) * 0.5 + 0.3
    return d, u, v


@pytest.mark.parametrize("dims,r,iso", [((16, 16, 16), 1, True), ((32, 24, 20), 2, True), ((40, 33), 3, False),
                                        ((20, 18, 16), 4, True),
                                        # K1 = 256: the fused kernel's x-split rows (two warps per row)
                                        ((256, 12, 10), 1, True), ((256, 7, 9), 2, False), ((256, 21, 5), 4, True)])
def test_diag_prox_f64_vs_oracle(dims, r, iso):
    d, u, v = _diag_problem(7, dims, r)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=v, w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05,
                           mode="iso" if iso else "aniso", box=W.BoxSet(0.0, np.inf))
    rep = D.solve(prob, eps=1e-300, max_iter=60)
    ref = O.fgp_prox(dims, v, O.Metric(U=u, d=d), reg=0.05, isotropic=iso, eps=1e-300, max_iter=60)
    assert rel_l2(rep.x, ref["x"]) <= F64_TOL
    assert rel_l2(rep.p_star, ref["p_star"]) <= F64_TOL
    assert rep.newton_iterations == ref["newton_iterations"]


@pytest.mark.parametrize("dims,r", [((32, 16, 12), 1), ((20, 18, 16), 2)])
def test_array_bounds_prox_f64_vs_oracle(dims, r):
    """Per-voxel box bounds (BoxSet with arrays, wpm.py:109-142): the general
    kernel serves them (the fused kernel takes scalar bounds only)."""
    d, u, v = _diag_problem(5, dims, r)
    rng = np.random.default_rng(6)
    n = int(np.prod(dims))
    lo = rng.uniform(-0.2, 0.1, n)
    hi = lo + rng.uniform(0.2, 1.0, n)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=v, w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05,
                           box=W.BoxSet(lo, hi))
    rep = D.solve(prob, eps=1e-300, max_iter=40)
    ref = O.fgp_prox(dims, v, O.Metric(U=u, d=d), reg=0.05, lo=lo, hi=hi, eps=1e-300, max_iter=40)
    assert rel_l2(rep.x, ref["x"]) <= F64_TOL
    assert rel_l2(rep.p_star, ref["p_star"]) <= F64_TOL
    assert np.all(rep.x >= lo) and np.all(rep.x <= hi)


def test_xsplit_rows_f32_vs_oracle():
    """K1 = 256 (x-split rows) in fp32 at a size with several row tiles and z segments."""
    d, u, v = _diag_problem(11, (256, 40, 24), 1)
    ref = O.fgp_prox((256, 40, 24), v, O.Metric(U=u, d=d), reg=0.05, eps=1e-300, max_iter=40)
    w = W.DiagPlusLowRank(1.0, torch.tensor(u, dtype=torch.float32, device="cuda"),
                          d=torch.tensor(d, dtype=torch.float32, device="cuda"))
    prob = D.DualTvProblem(grid=bq.Grid((256, 40, 24)), v=torch.tensor(v, dtype=torch.float32, device="cuda"), w=w,
                           reg=0.05)
    rep = D.solve(prob, eps=1e-300, max_iter=40)
    assert rel_l2(rep.x.double().cpu().numpy(), ref["x"]) <= F32_TOL
    assert rel_l2(rep.p_star.double().cpu().numpy(), ref["p_star"]) <= F32_TOL


@pytest.mark.parametrize("dims,r", [((128, 36, 20), 1), ((128, 30, 18), 2), ((256, 20, 16), 1), ((256, 18, 12), 2)])
def test_scalar_tau_f32_stage_ring_vs_oracle(dims, r):
    """fp32 BQNPM metric tau I + U U^T at ranks 1-2: the fused kernel's 3-deep
    stage ring (K1 = 128, and K1 = 256 x-split rows where it fits)."""
    rng = np.random.default_rng(21)
    n = int(np.prod(dims))
    u = rng.standard_normal((n, r)) / np.sqrt(n)
    v = rng.standard_normal(n) + 0.5
    ref = O.fgp_prox(dims, v, O.Metric(U=u, tau=1.25), reg=0.05, eps=1e-300, max_iter=40)
    w = W.DiagPlusLowRank(1.25, torch.tensor(u, dtype=torch.float32, device="cuda"))
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=torch.tensor(v, dtype=torch.float32, device="cuda"), w=w,
                           reg=0.05, box=W.BoxSet(0.0, np.inf))
    rep = D.solve(prob, eps=1e-300, max_iter=40)
    assert rel_l2(rep.x.double().cpu().numpy(), ref["x"]) <= F32_TOL
    assert rel_l2(rep.p_star.double().cpu().numpy(), ref["p_star"]) <= F32_TOL


def test_config2_shape_f32_vs_f64_and_oracle_64():
    """Config-2 law (W = diag(d) + uu^T, iso TV 0.05, box [0, inf), 100 FGP iters)
    at 64^3: fp32 and fp64 device results vs the fp64 oracle."""
    from paper_2307_02043_b200.configs import config2_inputs

    inp = config2_inputs(n=64)
    ref = O.fgp_prox((64, 64, 64), inp["v"], O.Metric(U=inp["u"][:, None], d=inp["d"]), reg=0.05,
                     eps=1e-300, max_iter=100)
    for dtype, tol in [(torch.float64, F64_TOL), (torch.float32, F32_TOL)]:
        w = W.DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=dtype, device="cuda"),
                              d=torch.tensor(inp["d"], dtype=dtype, device="cuda"))
        v = torch.tensor(inp["v"], dtype=dtype, device="cuda")
        rep = D.solve(D.DualTvProblem(grid=bq.Grid((64, 64, 64)), v=v, w=w, reg=0.05), eps=1e-300, max_iter=100)
        assert rel_l2(rep.x.double().cpu().numpy(), ref["x"]) <= tol
        assert rel_l2(rep.p_star.double().cpu().numpy(), ref["p_star"]) <= tol


def test_prox_is_deterministic():
    d, u, v = _diag_problem(3, (32, 32, 32), 2)
    prob = D.DualTvProblem(grid=bq.Grid((32, 32, 32)), v=torch.tensor(v, device="cuda"),
                           w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05)
    a = D.solve(prob, eps=1e-300, max_iter=50)
    b = D.solve(prob, eps=1e-300, max_iter=50)
    assert torch.equal(a.x, b.x) and torch.equal(a.p_star, b.p_star)


@pytest.mark.parametrize("dims,r,dtype", [((64, 64, 64), 1, torch.float32), ((48, 40, 36), 2, torch.float64),
                                          ((128, 128, 40), 1, torch.float32)])
def test_compact_near_list_is_bit_identical_to_the_gather(monkeypatch, dims, r, dtype):
    """Short near lists reach the on-chip Newton through the grid-wide compact
    copy (atomic slot reservation, sorted back into segment order) instead of
    the count scan + gather: same entries in the same order, so x, P* and the
    Newton counts are bit-identical with the compact copy switched off."""
    d, u, v = _diag_problem(11, dims, r)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=torch.tensor(v, dtype=dtype, device="cuda"),
                           w=W.DiagPlusLowRank(1.0, torch.tensor(u, dtype=dtype, device="cuda"),
                                               d=torch.tensor(d, dtype=dtype, device="cuda")), reg=0.05)
    a = D.solve(prob, eps=1e-300, max_iter=80)
    monkeypatch.setenv("BQ_PROX_NOCL", "1")
    b = D.solve(prob, eps=1e-300, max_iter=80)
    assert a.newton_iterations == b.newton_iterations and a.iterations == b.iterations == 80
    assert torch.equal(a.x, b.x) and torch.equal(a.p_star, b.p_star)


def test_headline_shape_is_bit_reproducible():
    """128^3 fp32 on all 148 blocks: the atomic slot reservations of the compact
    near list run in a different order every time; x and P* must not depend on it."""
    from paper_2307_02043_b200.configs import config2_inputs

    inp = config2_inputs(n=128)
    w = W.DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=torch.float32, device="cuda"),
                          d=torch.tensor(inp["d"], dtype=torch.float32, device="cuda"))
    prob = D.DualTvProblem(grid=bq.Grid((128, 128, 128)), v=torch.tensor(inp["v"], dtype=torch.float32, device="cuda"),
                           w=w, reg=0.05)
    first = D.solve(prob, eps=1e-300, max_iter=60)
    for _ in range(4):
        again = D.solve(prob, eps=1e-300, max_iter=60)
        assert again.newton_iterations == first.newton_iterations
        assert torch.equal(again.x, first.x) and torch.equal(again.p_star, first.p_star)


def test_per_tile_block_assignment_matches_contiguous_split(monkeypatch):
    """128-voxel rows over 148 blocks: the per-tile z-segments against one
    contiguous split of the tile-plane sequence (different partial-sum
    grouping only)."""
    dims = (128, 128, 48)
    d, u, v = _diag_problem(12, dims, 1)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=torch.tensor(v, device="cuda"),
                           w=W.DiagPlusLowRank(1.0, torch.tensor(u, device="cuda"), d=torch.tensor(d, device="cuda")),
                           reg=0.05)
    a = D.solve(prob, eps=1e-300, max_iter=40)
    monkeypatch.setenv("BQ_PROX_TILEBLK", "0")
    b = D.solve(prob, eps=1e-300, max_iter=40)
    assert a.newton_iterations == b.newton_iterations
    assert rel_l2(a.x.cpu().numpy(), b.x.cpu().numpy()) <= 1e-12
    assert rel_l2(a.p_star.cpu().numpy(), b.p_star.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("i", range(4))
def test_wpm_box_matches_reference_golden(golden, i):
    w = W.DiagPlusLowRank(float(golden[f"wpm{i}_tau"]), golden[f"wpm{i}_U"])
    beta0 = golden[f"wpm{i}_beta0"] if bool(golden[f"wpm{i}_has_beta0"]) else None
    u, info = W.wpm_box(golden[f"wpm{i}_x"], w, W.BoxSet(float(golden[f"wpm{i}_lo"]), float(golden[f"wpm{i}_hi"])),
                        beta0=beta0, full_output=True)
    assert rel_l2(u, golden[f"wpm{i}_u"]) <= F64_TOL
    bref = golden[f"wpm{i}_beta"]
    assert np.max(np.abs(info["beta"] - bref)) <= 1e-8 * max(1.0, float(np.max(np.abs(bref))))
    assert info["iterations"] == int(golden[f"wpm{i}_iters"])


@pytest.mark.parametrize("i", range(5))
def test_metric_matches_reference_golden(golden, i):
    w = W.DiagPlusLowRank(float(golden[f"metric{i}_tau"]), golden[f"metric{i}_U"], sign=int(golden[f"metric{i}_sign"]))
    x = golden[f"metric{i}_x"]
    assert rel_l2(W.apply_metric(w, x), golden[f"metric{i}_Wx"]) <= 1e-13
    assert rel_l2(W.apply_metric_inverse(w, x), golden[f"metric{i}_Winvx"]) <= 1e-12


def test_metric_errors_map_to_value_error():
    with pytest.raises(ValueError):
        W.DiagPlusLowRank(0.0, np.zeros((3, 0)))
    with pytest.raises(ValueError):
        W.DiagPlusLowRank(1.0, np.array([[2.0], [0.0]]), sign=-1)
    W.DiagPlusLowRank(1.0, 0.4 * np.array([[2.0], [0.0]]), sign=-1)
    w = W.DiagPlusLowRank(1.0, np.ones((4, 1)))
    with pytest.raises(ValueError):
        W.apply_metric(w, np.ones(5))


def test_solve_rejects_bad_arguments():
    rng = np.random.default_rng(15)
    prob = D.DualTvProblem(grid=bq.Grid((8, 8)), v=rng.standard_normal(64),
                           w=W.DiagPlusLowRank(1.0, rng.standard_normal((64, 1)) / 8), reg=0.3)
    with pytest.raises(ValueError):
        D.solve(prob, eps=0.0)
    with pytest.raises(ValueError):
        D.solve(prob, max_iter=0)
    with pytest.raises(ValueError):
        D.DualTvProblem(grid=prob.grid, v=prob.v, w=prob.w, reg=-1.0)


def test_tv_value_matches_reference_golden(golden):
    for key in ["7", "5x4", "4x3x2", "6x5x4"]:
        dims = tuple(int(k) for k in key.split("x"))
        x = golden[f"stencil_{key}_x"]
        assert bq.tv_value(bq.Grid(dims), x, "iso") == pytest.approx(float(golden[f"stencil_{key}_tv_iso"]), rel=1e-13)
        assert bq.tv_value(bq.Grid(dims), x, "aniso") == pytest.approx(float(golden[f"stencil_{key}_tv_aniso"]),
                                                                        rel=1e-13)


@pytest.mark.parametrize("dims,r,dtype,tol", [((256, 256, 72), 4, torch.float64, 1e-9),
                                              ((256, 256, 256), 1, torch.float32, 1e-4)])
def test_large_grid_fused_matches_general_kernel(monkeypatch, dims, r, dtype, tol):
    """Grids large enough for the scaled near-list capacity (> 64 entries per warp)
    and the x-split rows: the fused kernel vs the general-shape kernel (itself
    pinned to the oracle above), same inputs, 30 FGP iterations."""
    n = int(np.prod(dims))
    g = torch.Generator(device="cuda").manual_seed(5)
    v = torch.randn(n, generator=g, device="cuda", dtype=dtype) * 0.5 + 0.3
    U = torch.randn(n, r, generator=g, device="cuda", dtype=dtype) / np.sqrt(n)
    d = torch.rand(n, generator=g, device="cuda", dtype=dtype) * 1.5 + 0.5
    w = W.DiagPlusLowRank(1.0, U, d=d) if r == 1 else W.DiagPlusLowRank(1.25, U)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=v, w=w, reg=0.05)
    fused = D.solve(prob, eps=1e-300, max_iter=30)
    monkeypatch.setenv("BQ_PROX_GENERAL", "1")
    general = D.solve(prob, eps=1e-300, max_iter=30)
    assert fused.iterations == general.iterations == 30
    assert rel_l2(fused.x.double().cpu().numpy(), general.x.double().cpu().numpy()) <= tol
    assert rel_l2(fused.p_star.double().cpu().numpy(), general.p_star.double().cpu().numpy()) <= tol


def test_mixed_dtype_inputs_compute_in_metric_dtype():
    """numpy (fp64) metric with a torch fp32 v: the arithmetic runs in the metric's
    dtype (U and d live there), the outputs come back in v's dtype."""
    d, u, v = _diag_problem(9, (24, 20, 16), 1)
    ref = O.fgp_prox((24, 20, 16), v, O.Metric(U=u, d=d), reg=0.05, eps=1e-300, max_iter=30)
    vt = torch.tensor(v, dtype=torch.float32, device="cuda")
    rep = D.solve(D.DualTvProblem(grid=bq.Grid((24, 20, 16)), v=vt, w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05),
                  eps=1e-300, max_iter=30)
    assert rep.x.dtype == torch.float32 and rep.p_star.dtype == torch.float32
    # v rounded to fp32 on input; everything after it in fp64
    ref32 = O.fgp_prox((24, 20, 16), vt.double().cpu().numpy(), O.Metric(U=u, d=d), reg=0.05, eps=1e-300,
                       max_iter=30)
    assert rel_l2(rep.x.double().cpu().numpy(), ref32["x"]) <= 1e-6
    assert rel_l2(rep.x.double().cpu().numpy(), ref["x"]) <= F32_TOL
    # fp32 metric with numpy (fp64) v: computes in fp32
    w32 = W.DiagPlusLowRank(1.0, torch.tensor(u, dtype=torch.float32, device="cuda"),
                            d=torch.tensor(d, dtype=torch.float32, device="cuda"))
    rep2 = D.solve(D.DualTvProblem(grid=bq.Grid((24, 20, 16)), v=v, w=w32, reg=0.05), eps=1e-300, max_iter=30)
    assert isinstance(rep2.x, np.ndarray)
    assert rel_l2(rep2.x, ref["x"]) <= F32_TOL
    # a workspace in another dtype than the metric is refused
    ws = D.ProxWorkspace(bq.Grid((24, 20, 16)), torch.float32, torch.device("cuda", 0))
    with pytest.raises(ValueError):
        D.solve_async(D.DualTvProblem(grid=bq.Grid((24, 20, 16)), v=vt, w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05),
                      ws)


def test_concurrent_streams_do_not_share_reduction_scratch():
    """A prox on a small grid (fewer blocks than SMs) on one stream and metric
    gram reductions on another stream of the same context run concurrently; each
    stream has its own partials / arrival counters, so both results are exact."""
    d, u, v = _diag_problem(13, (32, 16, 8), 2)
    prob = D.DualTvProblem(grid=bq.Grid((32, 16, 8)), v=torch.tensor(v, device="cuda"),
                           w=W.DiagPlusLowRank(1.0, u, d=d), reg=0.05)
    solo = D.solve(prob, eps=1e-300, max_iter=80)
    g = torch.Generator(device="cuda").manual_seed(3)
    U2 = torch.randn(1 << 20, 4, generator=g, device="cuda", dtype=torch.float64) / 1024.0
    w_solo = W.DiagPlusLowRank(2.0, U2)
    side = torch.cuda.Stream()
    grams = []
    ws = D.ProxWorkspace(prob.grid, torch.float64, torch.device("cuda", 0))
    torch.cuda.synchronize()
    D.solve_async(prob, ws, eps=1e-300, max_iter=80)
    with torch.cuda.stream(side):
        for _ in range(20):
            grams.append(W.DiagPlusLowRank(2.0, U2).gram.clone())
    torch.cuda.synchronize()
    assert torch.equal(ws.x, solo.x) and torch.equal(ws.p, solo.p_star)
    for gr in grams:
        assert torch.equal(gr, w_solo.gram)


def test_default_omega_for_negative_sign_diag_metric():
    """W = diag(d) - u u^T: omega defaults to 1/(min(d) (1 - lambda_max(U^T D^-1 U))),
    a valid bound on 1/lambda_min(W) (1/min(d) is not), and the solve converges."""
    rng = np.random.default_rng(4)
    n = 12 * 10 * 8
    d = rng.uniform(0.5, 2.0, n)
    u = rng.standard_normal((n, 1)) * 0.6 / np.sqrt(n / 2.0)
    w = W.DiagPlusLowRank(1.0, u, sign=-1, d=d)
    lam_min = np.linalg.eigvalsh(w.dense())[0]
    assert w.default_omega() >= 1.0 / lam_min * (1 - 1e-12)
    assert w.default_omega() > 1.0 / d.min()
    v = rng.standard_normal(n)
    prob = D.DualTvProblem(grid=bq.Grid((12, 10, 8)), v=v, w=w, reg=0.05)
    rep = D.solve(prob, eps=1e-8, max_iter=2000)
    ref = O.fgp_prox((12, 10, 8), v, O.Metric(U=u, d=d, sign=-1), reg=0.05, eps=1e-8, max_iter=2000,
                     omega=prob.omega)
    assert rep.converged and ref["converged"] and rep.iterations == ref["iterations"]
    assert rel_l2(rep.x, ref["x"]) <= F64_TOL

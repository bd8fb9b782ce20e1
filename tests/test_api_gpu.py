"""The rest of the reference's public hot-path API on the device: standalone TV
stencils (tv_ops.py:107-225), phi / Newton matrix / semismooth_newton /
moreau_envelope (wpm.py:150-260), the dual-solver helpers
(dual_tv_solver.py:95-152, 253-260) and the physics views' ViewProblem
surface (forward_models.py:43-83).  Checked against the reference golden
vectors and the CPU oracle."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import prox as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200 import tv_ops as T  # noqa: E402
from paper_2307_02043_b200 import wpm as W  # noqa: E402

KEYS = ["7", "5x4", "4x3x2", "6x5x4"]


@pytest.mark.parametrize("key", KEYS)
def test_stencils_match_reference_golden(golden, key):
    dims = tuple(int(k) for k in key.split("x"))
    g = bq.Grid(dims)
    x = golden[f"stencil_{key}_x"]
    p = golden[f"stencil_{key}_p"]
    gs = T.gradient_stack(g, x)
    assert gs.shape == (g.ndim, g.size)
    assert rel_l2(gs, golden[f"stencil_{key}_grad"]) <= 1e-15
    assert T.dual_adjoint is T.gradient_stack
    for n in range(1, g.ndim + 1):
        assert rel_l2(T.apply_diff(g, x, n), golden[f"stencil_{key}_grad"][n - 1]) <= 1e-15
    assert rel_l2(T.dual_divergence(g, p), golden[f"stencil_{key}_div"]) <= 1e-15
    # the golden projects 2 P (make_golden.py), so that some columns leave the ball
    assert rel_l2(T.project_dual(2.0 * p, "iso"), golden[f"stencil_{key}_proj_iso"]) <= 1e-15
    assert rel_l2(T.project_dual(2.0 * p, "aniso"), golden[f"stencil_{key}_proj_aniso"]) <= 1e-15
    # the adjoint pair and the duality pairing (tv_ops.py:223-225)
    rng = np.random.default_rng(1)
    y = rng.standard_normal(g.size)
    for n in range(1, g.ndim + 1):
        lhs = float(T.apply_diff(g, x, n) @ y)
        rhs = float(x @ T.apply_diff_adjoint(g, y, n))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
        np.testing.assert_allclose(T.apply_diff_adjoint(g, y, n), O.diff_adjoint(dims, y, n), rtol=0, atol=1e-15)
    assert T.dual_pairing(g, p, x) == pytest.approx(float(np.sum(p * T.gradient_stack(g, x))), rel=1e-12)


def test_stencil_errors_and_torch_flavour():
    g = bq.Grid((6, 5, 4))
    with pytest.raises(ValueError):
        T.apply_diff(g, np.zeros(g.size), 4)
    with pytest.raises(ValueError):
        T.dual_divergence(g, np.zeros((2, g.size)))
    x = torch.randn(g.size, dtype=torch.float32, device="cuda")
    out = T.gradient_stack(g, x)
    assert isinstance(out, torch.Tensor) and out.dtype == torch.float32 and out.shape == (3, g.size)
    ref = O.grad(g.dims, x.double().cpu().numpy())
    assert rel_l2(out.double().cpu().numpy(), ref) <= 1e-6


def test_diff_operator_norm_and_maximizing_field():
    g = bq.Grid((12, 10, 8))
    lam = T.diff_operator_norm_sq(g, iters=200, seed=0)
    assert 0.8 * T.power_upper_bound(g) < lam <= T.power_upper_bound(g)
    rng = np.random.default_rng(2)
    x = rng.standard_normal(g.size)
    for mode in ("iso", "aniso"):
        f = T.tv_maximizing_field(g, x, mode)
        # <d(F), x> = <F, grad x> = TV(x) for the maximizing field
        assert T.dual_pairing(g, f, x) == pytest.approx(bq.tv_value(g, x, mode), rel=1e-12)


def _metric(rng, n, r, d=False, sign=1):
    U = rng.standard_normal((n, r)) * (0.3 / np.sqrt(n))
    if d:
        dv = rng.uniform(0.5, 2.0, n)
        return W.DiagPlusLowRank(1.0, U, sign=sign, d=dv), O.Metric(U=U, d=dv, sign=sign)
    return W.DiagPlusLowRank(1.3, U, sign=sign), O.Metric(tau=1.3, U=U, sign=sign)


@pytest.mark.parametrize("r,d,sign", [(1, False, 1), (3, False, -1), (2, True, 1)])
def test_phi_and_newton_matrix(r, d, sign):
    rng = np.random.default_rng(r)
    n = 500
    w, wo = _metric(rng, n, r, d, sign)
    x = rng.standard_normal(n)
    beta = rng.standard_normal(r) * 0.2
    box = W.BoxSet(-0.3, 0.8)
    z = x - sign * ((wo.U @ beta) / (wo.d if d else wo.tau))
    q = np.clip(z, -0.3, 0.8)
    ref = wo.U.T @ (x - q) + beta
    np.testing.assert_allclose(W.phi(beta, x, w, box), ref, rtol=1e-12, atol=1e-14)
    ins = (z > -0.3) & (z < 0.8)
    ua = wo.U[ins]
    h = np.eye(r) + sign * (ua.T @ (ua / (wo.d[ins][:, None] if d else wo.tau)))
    np.testing.assert_allclose(W.newton_matrix(beta, x, w, box), h, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("i", range(4))
def test_semismooth_newton_and_moreau_envelope_golden(golden, i):
    w = W.DiagPlusLowRank(float(golden[f"wpm{i}_tau"]), golden[f"wpm{i}_U"])
    box = W.BoxSet(float(golden[f"wpm{i}_lo"]), float(golden[f"wpm{i}_hi"]))
    x = golden[f"wpm{i}_x"]
    beta0 = golden[f"wpm{i}_beta0"] if bool(golden[f"wpm{i}_has_beta0"]) else None
    beta, info = W.semismooth_newton(x, w, box, beta0=beta0, full_output=True)
    bref = golden[f"wpm{i}_beta"]
    assert np.max(np.abs(beta - bref)) <= 1e-8 * max(1.0, float(np.max(np.abs(bref))))
    assert info["iterations"] == int(golden[f"wpm{i}_iters"])
    u = golden[f"wpm{i}_u"]
    wd = w.dense()
    env = 0.5 * float((u - x) @ wd @ (u - x))
    assert W.moreau_envelope(x, w, box, beta0=beta0) == pytest.approx(env, rel=1e-10)
    assert np.linalg.norm(W.phi(beta, x, w, box)) <= max(1e-6, info["residual"] * (1 + 1e-9))


def test_dual_helpers_match_oracle():
    rng = np.random.default_rng(5)
    dims = (10, 9, 8)
    n = int(np.prod(dims))
    U = rng.standard_normal((n, 2)) / np.sqrt(n)
    v = rng.standard_normal(n) + 0.3
    w = W.DiagPlusLowRank(1.4, U)
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=v, w=w, reg=0.07, box=W.BoxSet(0.0, 1.0))
    p = rng.standard_normal((3, n)) * 0.3
    wo = O.Metric(tau=1.4, U=U)
    wp_ref = v - 0.07 * wo.inverse(O.div(dims, p))
    wp = D.w_of_p(prob, p)
    assert rel_l2(wp, wp_ref) <= 1e-12
    q_ref, _ = O.wpm_box(wp_ref, wo, 0.0, 1.0)
    assert rel_l2(D.dual_gradient(prob, p), -2 * 0.07 * O.grad(dims, q_ref)) <= 1e-10
    wd = w.dense()
    obj_ref = float(wp_ref @ wd @ wp_ref - (wp_ref - q_ref) @ wd @ (wp_ref - q_ref))
    assert D.dual_objective(prob, p) == pytest.approx(obj_ref, rel=1e-10)
    x = np.clip(v, 0.0, 1.0)
    pobj = 0.5 * float((x - v) @ wd @ (x - v)) + 0.07 * O.tv_value(dims, x)
    assert D.primal_objective(prob, x) == pytest.approx(pobj, rel=1e-12)
    # a solved prox: primal = dual certificate gap small
    rep = D.solve(prob, eps=1e-300, max_iter=400)
    assert D.primal_objective(prob, rep.x) <= pobj
    lam_min = np.linalg.eigvalsh(wd)[0]
    assert D.metric_min_eig_inverse(w, iters=50) == pytest.approx(1.0 / lam_min, rel=1e-6)


def test_scatter_view_problem_surface():
    """jacobian_vec / adjoint_vec / value / gradient / self_check of the physics
    views (forward_models.py:43-83), Born and LS, c128 and c64."""
    from oracle import physics as P
    from paper_2307_02043_b200 import physics as PH

    s = P.Setup(n=10, n_views=3)
    x = P.ellipsoid_phantom(10, 3, 0.02, 0.06, seed=2)
    rng = np.random.default_rng(4)
    dx = rng.standard_normal(1000)
    for model in ("born", "ls"):
        om = P.ScatterModel(s, model, tol=1e-13, max_iter=400)
        views, vs = PH.make_scatter_views(10, 3, model=model, x_gt=x, dtype=torch.complex128, tol=1e-13,
                                          max_iter=400, batch=3, self_check=True)
        assert rel_l2(views[1].jacobian_vec(0.5 * x, dx), om.jvp(0.5 * x, 1, dx)) <= 1e-10
        views[2].self_check(1000, np.random.default_rng(7))
        assert isinstance(views[0].jacobian_vec(x, dx), np.ndarray)
    views32, _ = PH.make_scatter_views(10, 3, model="ls", x_gt=x, dtype=torch.complex64, tol=1e-6, batch=3)
    views32[0].self_check(1000, np.random.default_rng(8))


def test_volume_format_from_and_to_device(tmp_path):
    """A device x (flat Fortran layout == C-order (K3, K2, K1) tensor) is written
    with one D2H copy and reads back as the reference's n-d array."""
    from pathlib import Path

    from paper_2307_02043_b200 import formats as F

    x = np.load(Path(__file__).parent / "golden" / "ref_formats.npz")["volume"]
    xt = torch.tensor(x.reshape(-1, order="F"), device="cuda").reshape(3, 4, 5)
    F.dump_volume(xt, tmp_path / "d.tvqnvol")
    ref = (Path(__file__).parent / "golden" / "ref_volume_5x4x3.tvqnvol").read_bytes()
    assert (tmp_path / "d.tvqnvol").read_bytes() == ref
    back = F.load_volume(tmp_path / "d.tvqnvol", device="cuda")
    assert back.is_cuda and torch.equal(back, xt.reshape(-1))

"""Pin the CPU oracle to the reference's own outputs (golden vectors made by
tests/golden/make_golden.py from the unmodified reference) and to the
reference tests' known-answer cases.  CPU only."""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import prox as O


def _dims(key):
    return tuple(int(k) for k in key.split("x"))


@pytest.mark.parametrize("key", ["7", "5x4", "4x3x2", "6x5x4"])
def test_stencils_match_reference(golden, key):
    dims = _dims(key)
    x = golden[f"stencil_{key}_x"]
    p = golden[f"stencil_{key}_p"]
    np.testing.assert_array_equal(O.grad(dims, x), golden[f"stencil_{key}_grad"])
    np.testing.assert_array_equal(O.div(dims, p), golden[f"stencil_{key}_div"])
    assert O.tv_value(dims, x, True) == pytest.approx(float(golden[f"stencil_{key}_tv_iso"]), rel=1e-14)
    assert O.tv_value(dims, x, False) == pytest.approx(float(golden[f"stencil_{key}_tv_aniso"]), rel=1e-14)
    np.testing.assert_array_equal(O.project_dual(2.0 * p, True), golden[f"stencil_{key}_proj_iso"])
    np.testing.assert_array_equal(O.project_dual(2.0 * p, False), golden[f"stencil_{key}_proj_aniso"])


def test_stencil_adjointness():
    rng = np.random.default_rng(0)
    for dims in [(9,), (6, 5), (5, 4, 3)]:
        n = int(np.prod(dims))
        x = rng.standard_normal(n)
        p = rng.standard_normal((len(dims), n))
        lhs = float(np.sum(O.grad(dims, x) * p))
        rhs = float(x @ O.div(dims, p))
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("i", range(5))
def test_metric_matches_reference(golden, i):
    w = O.Metric(tau=float(golden[f"metric{i}_tau"]), U=golden[f"metric{i}_U"], sign=int(golden[f"metric{i}_sign"]),
                 n=golden[f"metric{i}_x"].size)
    x = golden[f"metric{i}_x"]
    assert rel_l2(w.apply(x), golden[f"metric{i}_Wx"]) < 1e-14
    assert rel_l2(w.inverse(x), golden[f"metric{i}_Winvx"]) < 1e-13


def test_metric_known_answers():
    # tests/test_wpm.py:62-64, :76-78 of the reference
    w = O.Metric(tau=1.0, U=np.array([[1.0], [0.0]]))
    np.testing.assert_allclose(w.apply([1.0, 1.0]), [2.0, 1.0])
    np.testing.assert_allclose(w.inverse([2.0, 1.0]), [1.0, 1.0])
    with pytest.raises(np.linalg.LinAlgError):
        O.Metric(tau=1.0, U=np.array([[2.0], [0.0]]), sign=-1)


@pytest.mark.parametrize("i", range(4))
def test_wpm_box_matches_reference(golden, i):
    x = golden[f"wpm{i}_x"]
    w = O.Metric(tau=float(golden[f"wpm{i}_tau"]), U=golden[f"wpm{i}_U"])
    beta0 = golden[f"wpm{i}_beta0"] if bool(golden[f"wpm{i}_has_beta0"]) else None
    u, info = O.wpm_box(x, w, float(golden[f"wpm{i}_lo"]), float(golden[f"wpm{i}_hi"]), beta0)
    assert rel_l2(u, golden[f"wpm{i}_u"]) < 1e-12
    assert rel_l2(info["beta"], golden[f"wpm{i}_beta"]) < 1e-10
    assert info["iterations"] == int(golden[f"wpm{i}_iters"])


def _prox_case(golden, i):
    k = f"prox{i}"
    dims = tuple(int(v) for v in golden[k + "_dims"])
    r = int(golden[k + "_rank"])
    n = int(np.prod(dims))
    w = O.Metric(tau=float(golden[k + "_tau"]), U=golden[k + "_U"] if r else None, n=n)
    warm = bool(golden[k + "_has_warm"])
    kw = dict(
        reg=float(golden[k + "_reg"]), lo=float(golden[k + "_lo"]), hi=float(golden[k + "_hi"]),
        isotropic=bool(golden[k + "_iso"]), eps=float(golden[k + "_eps"]),
        max_iter=int(golden[k + "_max_iter"]), accelerated=bool(golden[k + "_acc"]),
        p0=golden[k + "_p0"] if warm else None, beta0=golden[k + "_b0"] if (warm and r) else None,
    )
    return dims, golden[k + "_v"], w, kw


@pytest.mark.parametrize("i", range(12))
def test_prox_matches_reference(golden, i):
    dims, v, w, kw = _prox_case(golden, i)
    rep = O.fgp_prox(dims, v, w, **kw)
    k = f"prox{i}"
    assert rel_l2(rep["x"], golden[k + "_x"]) < 1e-12
    assert rel_l2(rep["p_star"], golden[k + "_p_star"]) < 1e-12
    assert rep["iterations"] == int(golden[k + "_iterations"])
    assert rep["converged"] == bool(golden[k + "_converged"])
    assert rep["newton_iterations"] == int(golden[k + "_newton"])
    assert rel_l2(rep["beta_star"], golden[k + "_beta"]) < 1e-10


@pytest.mark.parametrize("i", range(3))
def test_diag_extension_vs_condat_vu(golden, i):
    """diag(d)+uu^T prox (not representable in the reference) is pinned by the
    reference's independent dense Condat-Vu oracle (tests/oracles.py:60-90)."""
    k = f"diag{i}"
    dims = tuple(int(v) for v in golden[k + "_dims"])
    d, u, v = golden[k + "_d"], golden[k + "_U"], golden[k + "_v"]
    iso = bool(golden[k + "_iso"])
    w = O.Metric(U=u, d=d)
    reg = float(golden[k + "_reg"])
    rep = O.fgp_prox(dims, v, w, reg=reg, isotropic=iso, eps=1e-12, max_iter=6000)
    ours = O.primal_objective(dims, v, w, reg, rep["x"], iso)
    ref = float(golden[k + "_obj_cv"])
    assert ours <= ref * (1 + 1e-4)
    assert abs(ours - ref) <= 1e-4 * abs(ref)
    assert np.all(rep["x"] >= 0)


def test_diag_extension_reduces_to_reference_at_constant_d(golden):
    dims, v, w, kw = _prox_case(golden, 0)
    wd = O.Metric(U=w.U, d=np.full(v.size, w.tau))
    a = O.fgp_prox(dims, v, w, **kw)
    b = O.fgp_prox(dims, v, wd, **kw)
    assert rel_l2(b["x"], a["x"]) < 1e-13
    assert rel_l2(b["p_star"], a["p_star"]) < 1e-13


def test_sr1_matches_reference(golden):
    for i in range(golden["sr1_s"].shape[0]):
        tau, u = O.estimate_sr1(golden["sr1_s"][i], golden["sr1_m"][i], 0.8, 1.7)
        assert tau == pytest.approx(float(golden["sr1_tau"][i]), rel=1e-14)
        assert (u is not None) == bool(golden["sr1_has_u"][i])
        if u is not None:
            assert rel_l2(u, golden["sr1_u"][i]) < 1e-13


def test_sr1_known_answer():
    # tests/test_hessian_sr1.py:8-14
    tau, u = O.estimate_sr1(np.array([1.0, 0.0]), np.array([1.0, 0.0]), 0.8, 1.0)
    assert tau == pytest.approx(0.8)
    np.testing.assert_allclose(u, [np.sqrt(0.2), 0.0], atol=1e-14)


def test_vk_matches_reference(golden):
    slots = []
    for t in range(4):
        u = golden[f"vk_u{t}"] if bool(golden[f"vk_has_u{t}"]) else None
        slots.append((golden[f"vk_x{t}"], golden[f"vk_g{t}"], float(golden[f"vk_tau{t}"]), u))
    w = O.aggregate(slots)
    assert w.tau == pytest.approx(float(golden["vk_tau_w"]), rel=1e-15)
    np.testing.assert_array_equal(w.U, golden["vk_U_w"])
    assert rel_l2(O.v_k(slots, w, 0.7), golden["vk_v"]) < 1e-13


def test_schedule_matches_reference(golden):
    tab = np.array([[O.kappa(k, t, 4) for t in range(1, 5)] for k in range(1, 13)])
    np.testing.assert_array_equal(tab, golden["kappa_table"])
    np.testing.assert_array_equal(np.concatenate(O.partition_views(30, 4)), golden["partition_equi_30_4"])
    np.testing.assert_array_equal(np.concatenate(O.partition_views(30, 4, "contiguous")),
                                  golden["partition_contig_30_4"])


# ---- masked-spectrum views (forward_models.py) ---------------------------
@pytest.mark.parametrize("tag,strength", [("lin", 0.0), ("nl", 0.1)])
def test_view_oracle_matches_reference(golden, tag, strength):
    from oracle import views as OV

    dims = tuple(int(v) for v in golden[f"views_{tag}_dims"])
    ys = golden[f"views_{tag}_y"]
    # masks are recovered from the reference's own mask law via the package helper
    from paper_2307_02043_b200.forward_models import spectrum_masks
    from paper_2307_02043_b200.tv_ops import Grid

    masks, _ = spectrum_masks(Grid(dims), ys.shape[0], 0.5)
    views = [OV.DctView(dims, masks[i], ys[i], strength) for i in range(ys.shape[0])]
    x = golden[f"views_{tag}_x"]
    assert rel_l2(views[0].forward(x), golden[f"views_{tag}_fwd0"]) < 1e-14
    np.testing.assert_allclose([v.value(x) for v in views], golden[f"views_{tag}_values"], rtol=1e-12)
    assert rel_l2(OV.subset_gradient(views, [1, 4, 6], x), golden[f"views_{tag}_grad_sub"]) < 1e-12
    # the package's phantom law reproduces the reference's
    from paper_2307_02043_b200.forward_models import make_phantom

    np.testing.assert_array_equal(make_phantom(Grid(dims), seed=3).values, golden[f"views_{tag}_phantom"])

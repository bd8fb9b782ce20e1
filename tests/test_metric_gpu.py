"""Device SR1 estimate, slot aggregation and v_k (through the C ABI) against the
reference golden vectors (tests/golden, made by the unmodified reference)."""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_02043_b200 import hessian_sr1 as H  # noqa: E402
from paper_2307_02043_b200 import metric_ops as M  # noqa: E402


def test_sr1_matches_reference_golden(golden):
    for i in range(golden["sr1_s"].shape[0]):
        est = H.estimate_sr1(golden["sr1_s"][i], golden["sr1_m"][i], gamma=0.8, alpha_fallback=1.7)
        assert est.tau == pytest.approx(float(golden["sr1_tau"][i]), rel=1e-12)
        assert (est.u is not None) == bool(golden["sr1_has_u"][i])
        if est.u is not None:
            assert rel_l2(est.u, golden["sr1_u"][i]) <= 1e-10


def test_sr1_known_answers_and_errors():
    # tests/test_hessian_sr1.py:8-31 of the reference
    est = H.estimate_sr1(np.array([1.0, 0.0]), np.array([1.0, 0.0]), gamma=0.8, alpha_fallback=1.0)
    assert est.tau == pytest.approx(0.8)
    np.testing.assert_allclose(est.u, [np.sqrt(0.2), 0.0], atol=1e-14)
    est = H.estimate_sr1(np.array([1.0]), np.array([-1.0]), gamma=0.8, alpha_fallback=7.0)
    assert est.tau == 7.0 and est.u is None
    est = H.estimate_sr1(np.array([1.0, 0.0]), np.array([0.0, 1.0]), gamma=0.8, alpha_fallback=3.0)
    assert est.tau == 3.0 and est.u is None
    with pytest.raises(ValueError):
        H.estimate_sr1(np.zeros(4), np.ones(4))
    with pytest.raises(ValueError):
        H.estimate_sr1(np.ones(3), np.ones(3), gamma=1.0)
    with pytest.raises(ValueError):
        H.estimate_sr1(np.ones(3), np.ones(3), alpha_fallback=0.0)


def test_sr1_secant_equation_f32():
    rng = np.random.default_rng(3)
    n = 4096
    a = rng.uniform(0.5, 2.0, n)
    s = rng.standard_normal(n)
    m = a * s
    st = torch.tensor(s, dtype=torch.float32, device="cuda")
    mt = torch.tensor(m, dtype=torch.float32, device="cuda")
    est = H.estimate_sr1(st, mt)
    if est.u is not None:
        bs = est.apply(st)
        assert rel_l2(bs.cpu().numpy(), m) < 1e-4


def test_vk_matches_reference_golden(golden):
    slots = []
    for t in range(4):
        u = golden[f"vk_u{t}"] if bool(golden[f"vk_has_u{t}"]) else None
        slots.append(M.SubsetSlot(x=golden[f"vk_x{t}"], grad=golden[f"vk_g{t}"],
                                  hess=H.Sr1Estimate(tau=float(golden[f"vk_tau{t}"]), u=u)))
    w = M.aggregate_metric(slots)
    assert w.tau == pytest.approx(float(golden["vk_tau_w"]), rel=1e-15)
    np.testing.assert_allclose(w.U, golden["vk_U_w"], rtol=0, atol=0)
    v = M.compute_v_k(slots, w, 0.7)
    assert rel_l2(v, golden["vk_v"]) <= 1e-12


def test_schedule_matches_reference_golden(golden):
    tab = np.array([[M.kappa(k, t, 4) for t in range(1, 5)] for k in range(1, 13)])
    np.testing.assert_array_equal(tab, golden["kappa_table"])
    np.testing.assert_array_equal(np.concatenate(M.partition_views(30, 4)), golden["partition_equi_30_4"])


def test_diag_metric_construction_checks():
    # DiagPlusLowRank with a per-voxel diagonal reads min(d) and the gram in one
    # device->host copy: d > 0 (NaN rejected too), W PD and omega = 1/min(d) (D-6)
    from paper_2307_02043_b200.wpm import DiagPlusLowRank

    rng = np.random.default_rng(11)
    n = 3000
    d = rng.uniform(0.5, 2.0, n)
    u = rng.standard_normal((n, 2)) / np.sqrt(n)
    w = DiagPlusLowRank(1.0, u, d=d, dtype=torch.float64)
    assert w.min_diag() == pytest.approx(d.min(), rel=0, abs=0)
    g = w.gram.cpu().numpy().reshape(2, 2)
    np.testing.assert_allclose(g, u.T @ (u / d[:, None]), rtol=1e-12)
    w0 = DiagPlusLowRank(1.0, np.zeros((n, 0)), d=d, dtype=torch.float64)  # rank 0: min(d) alone
    assert w0.rank == 0 and w0.min_diag() == pytest.approx(d.min(), rel=0, abs=0)
    for bad in (0.0, -1.0, np.nan):
        db = d.copy()
        db[n // 3] = bad
        with pytest.raises(ValueError, match="positive"):
            DiagPlusLowRank(1.0, u, d=db, dtype=torch.float64)
    big = np.zeros((n, 1))
    big[0, 0] = 10.0  # I - U^T D^-1 U / 1 is not PD
    with pytest.raises(ValueError, match="positive definite"):
        DiagPlusLowRank(1.0, big, sign=-1, d=d, dtype=torch.float64)


def test_compute_v_k_rejects_per_voxel_diagonal():
    """bq_vk has no d: a per-voxel metric is refused instead of dividing by tau = 0."""
    from paper_2307_02043_b200.wpm import DiagPlusLowRank

    n = 64
    rng = np.random.default_rng(2)
    slots = [M.SubsetSlot(x=rng.standard_normal(n), grad=rng.standard_normal(n), hess=H.Sr1Estimate(tau=1.0))]
    w = DiagPlusLowRank(1.0, rng.standard_normal((n, 1)) / 8, d=rng.uniform(0.5, 2, n))
    with pytest.raises(ValueError):
        M.compute_v_k(slots, w, 1.0)


def test_metric_check_min_and_gram_and_nan():
    """bq_metric_check (DiagPlusLowRank's one-pass validation): min(d), the gram,
    and a NaN in d rejected like the reference's (d > 0).all()."""
    from paper_2307_02043_b200.wpm import DiagPlusLowRank

    rng = np.random.default_rng(8)
    n = 100_003
    d = rng.uniform(0.5, 2.0, n)
    U = rng.standard_normal((n, 3)) / np.sqrt(n)
    w = DiagPlusLowRank(1.0, U, d=d)
    assert w.min_diag() == d.min()
    np.testing.assert_allclose(w.gram.reshape(3, 3).cpu().numpy(), U.T @ (U / d[:, None]), rtol=1e-12)
    w2 = DiagPlusLowRank(1.7, U)
    np.testing.assert_allclose(w2.gram.reshape(3, 3).cpu().numpy(), U.T @ U, rtol=1e-12)
    d[77] = np.nan
    with pytest.raises(ValueError):
        DiagPlusLowRank(1.0, U, d=d)
    d[77] = -1.0
    with pytest.raises(ValueError):
        DiagPlusLowRank(1.0, U, d=d)

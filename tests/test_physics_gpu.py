"""Device Born / Lippmann-Schwinger views against the builder-specified CPU
oracle (oracle/physics.py; parity unpinned w.r.t. the reference, which has no
physics -- SURVEY F2).  c128 <= 1e-10 with converged solves, c64 <= 1e-4."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import physics as P

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_02043_b200 import physics as PH  # noqa: E402


def _setup(n=12, L=6):
    return P.Setup(n=n, n_views=L), P.ellipsoid_phantom(n, 4, 0.02, 0.08, seed=7)


@pytest.mark.parametrize("model", ["born", "ls"])
def test_forward_matches_oracle_c128(model):
    s, x = _setup()
    om = P.ScatterModel(s, model, tol=1e-13, max_iter=400)
    vs = PH.ScatterViewSet(s.n, s.n_views, model=model, dtype=torch.complex128, tol=1e-13, max_iter=400, batch=4)
    xt = torch.tensor(x, device="cuda")
    got = vs.forward(xt, [0, 1, 2, 3, 4, 5]).cpu().numpy()
    for l in range(s.n_views):
        assert rel_l2(got[l], om.forward(x, l)) <= 1e-10


@pytest.mark.parametrize("model", ["born", "ls"])
def test_subset_gradient_matches_oracle_c128(model):
    s, x = _setup()
    om = P.ScatterModel(s, model, tol=1e-13, max_iter=400)
    vs = PH.ScatterViewSet(s.n, s.n_views, model=model, dtype=torch.complex128, tol=1e-13, max_iter=400, batch=4)
    ys = np.array([om.forward(0.7 * x, l) for l in range(s.n_views)])
    vs.y.copy_(torch.tensor(ys, device="cuda"))
    idx = [0, 2, 3, 5, 1]
    g = vs.subset_gradient(idx, torch.tensor(x, device="cuda")).cpu().numpy()
    gref = sum(om.gradient(x, l, ys[l]) for l in idx) / len(idx)
    assert rel_l2(g, gref) <= 1e-10
    c = vs.costs(idx, torch.tensor(x, device="cuda")).cpu().numpy()
    np.testing.assert_allclose(c, [om.value(x, l, ys[l]) for l in idx], rtol=1e-10)


def test_ls_c64_close_to_oracle_and_iteration_counts():
    s, x = _setup(n=16, L=4)
    om = P.ScatterModel(s, "ls", tol=1e-6, max_iter=500)
    vs = PH.ScatterViewSet(s.n, s.n_views, model="ls", dtype=torch.complex64, tol=1e-6, max_iter=500, batch=4)
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")
    got = vs.forward(xt, [0, 1, 2, 3]).cpu().numpy()
    for l in range(4):
        assert rel_l2(got[l], om.forward(x, l)) <= 1e-4
    # BiCGSTAB iteration counts agree with the oracle within one iteration
    assert max(abs(a - b) for a, b in zip(vs.iters_forward[-4:], om.last_iters[-4:])) <= 1


def test_device_adjoint_identity():
    s, x = _setup(n=10, L=3)
    vs = PH.ScatterViewSet(s.n, s.n_views, model="ls", dtype=torch.complex128, tol=1e-13, max_iter=400, batch=3)
    om = P.ScatterModel(s, "ls", tol=1e-13, max_iter=400)
    rng = np.random.default_rng(3)
    dx = rng.standard_normal(s.n ** 3)
    rr = rng.standard_normal(2 * s.n ** 2)
    view = PH.ScatterView(vs, 1)
    lhs = float(om.jvp(x, 1, dx) @ rr)
    rhs = float(dx @ view.adjoint_vec(x, rr))
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))


def test_batched_equals_unbatched():
    s, x = _setup(n=12, L=5)
    xt = torch.tensor(x, device="cuda")
    a = PH.ScatterViewSet(s.n, 5, model="ls", dtype=torch.complex128, tol=1e-12, batch=5)
    b = PH.ScatterViewSet(s.n, 5, model="ls", dtype=torch.complex128, tol=1e-12, batch=1)
    fa = a.forward(xt, [0, 1, 2, 3, 4]).cpu().numpy()
    fb = np.concatenate([b.forward(xt, [l]).cpu().numpy() for l in range(5)])
    assert rel_l2(fa, fb) <= 1e-12


def test_config1_bqnpm_matches_reference_loop():
    """BASELINE config 1 end to end (first Born, 32^3, c128, L=16, K_s=4, 20 outer
    iterations, lambda 1e-3, box [0, 0.1]): the device BQNPM loop on device Born
    views vs the REFERENCE bqnpm_run driving the CPU Born oracle
    (tests/golden/config1_golden.npz).  North star: reconstruction <= 1e-3."""
    from pathlib import Path

    from paper_2307_02043_b200 import solvers as S
    from paper_2307_02043_b200.tv_ops import Grid
    from paper_2307_02043_b200.wpm import BoxSet

    z = np.load(Path(__file__).parent / "golden" / "config1_golden.npz")
    views, vs = PH.make_scatter_views(32, 16, model="born", dtype=torch.complex128, theta_deg=35.0, batch=8)
    vs.y.copy_(torch.tensor(z["c1_y"], device="cuda"))
    grid = Grid((32, 32, 32))
    box = BoxSet(0.0, 0.1)
    x0 = S.scaled_adjoint_initializer(views, grid, box)
    assert rel_l2(x0.cpu().numpy(), z["c1_x0"]) <= 1e-10
    x0r = S.default_initializer(views, grid, box)  # the reference initializer (saturates at the box bound)
    assert rel_l2(x0r.cpu().numpy(), z["c1_x0_reference_initializer"]) <= 1e-10
    al = S.estimate_subset_lipschitz(views, S.partition_views(16, 4), x0, 30, 1.05, 0)
    np.testing.assert_allclose(al, z["c1_alphas"], rtol=1e-9)
    cfg = S.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=20, box=box, seed=0, alphas=z["c1_alphas"])
    x, tr = S.bqnpm_run(views, grid, cfg, x0=z["c1_x0"], ground_truth=z["c1_xgt"])
    assert rel_l2(x, z["c1_x"]) <= 1e-3
    assert rel_l2(x, z["c1_x"]) <= 1e-8  # measured: far inside the north-star bound
    np.testing.assert_allclose(tr.column("cost"), z["c1_cost"], rtol=1e-8)
    np.testing.assert_array_equal(tr.column("inner_iters"), z["c1_inner"])
    # the run reconstructs: SNR of dn rises from the initial guess (3.7 dB) to 7.4 dB
    snr = tr.column("snr_db")
    np.testing.assert_allclose(snr, z["c1_snr"], atol=1e-6)
    assert snr[-1] > snr[0] + 3.0 > 3.0


def test_config3_law_ls_bqnpm_matches_reference_loop():
    """Config-3 law at reduced size (LS, n=20 padded to 40^3, L=8, K_s=4, 4 outer
    iterations): the device BQNPM loop on device LS views (BiCGSTAB to 1e-12)
    vs the REFERENCE bqnpm_run driving the CPU LS oracle."""
    from pathlib import Path

    from paper_2307_02043_b200 import solvers as S
    from paper_2307_02043_b200.tv_ops import Grid
    from paper_2307_02043_b200.wpm import BoxSet

    z = np.load(Path(__file__).parent / "golden" / "config3s_golden.npz")
    views, vs = PH.make_scatter_views(20, 8, model="ls", dtype=torch.complex128, theta_deg=35.0, batch=4,
                                      tol=1e-12, max_iter=1000)
    vs.y.copy_(torch.tensor(z["c3_y"], device="cuda"))
    grid = Grid((20, 20, 20))
    box = BoxSet(0.0, 0.1)
    x0 = S.default_initializer(views, grid, box)
    assert rel_l2(x0.cpu().numpy(), z["c3_x0"]) <= 1e-10
    al = S.estimate_subset_lipschitz(views, S.partition_views(8, 4), x0, 10, 1.05, 0)
    np.testing.assert_allclose(al, z["c3_alphas"], rtol=1e-8)
    cfg = S.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=4, box=box, seed=0, alphas=z["c3_alphas"])
    x, tr = S.bqnpm_run(views, grid, cfg, x0=z["c3_x0"])
    assert rel_l2(x, z["c3_x"]) <= 1e-3
    assert rel_l2(x, z["c3_x"]) <= 1e-7
    np.testing.assert_allclose(tr.column("cost"), z["c3_cost"], rtol=1e-7)

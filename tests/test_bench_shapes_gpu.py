"""Parity on the exact shapes bench.py measures, against oracle / reference
fixtures made by tests/golden/make_bench_fixtures.py.

* config 2: 128^3 fp32, W = diag(d) + u u^T, 100 FGP iterations -- the
  headline kernel wtv_fused_kernel<float, 1, 128> -- vs the fp64 port (<= 1e-4),
  its fp64 twin (<= 1e-10, same Newton count), and the scalar-tau twin vs the
  UNMODIFIED reference solve (<= 1e-10 fp64, <= 1e-4 fp32).
* config 4: n = 128 complex64 (pruned passes at m = 256): a 2-view subset
  gradient (<= 1e-4) and a fixed-K BiCGSTAB solve (<= 1e-4) vs the c128 oracle.
* config 3 law at n = 64 (pruned passes at m = 128): the device BQNPM loop vs the
  reference bqnpm_run driving the oracle, 3 outer iterations (<= 1e-3, north star).

128^3 vectors are compared on the fixture's strided sample (relative L2) and
through whole-vector summaries (norm, sum, seeded +/-1 probe)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200 import physics as PH  # noqa: E402
from paper_2307_02043_b200 import solvers as S  # noqa: E402
from paper_2307_02043_b200 import wpm as W  # noqa: E402
from paper_2307_02043_b200.configs import config2_inputs, ls_phantom  # noqa: E402

GOLD = Path(__file__).parent / "golden"
STRIDE, PROBE_SEED = 17, 99


def _probe(n):
    return np.random.default_rng(PROBE_SEED).integers(0, 2, n).astype(float) * 2.0 - 1.0


def check_summary(z, prefix, got, tol, stride=STRIDE):
    """Strided-sample relative L2 <= tol, |norm| and |sum| relative <= tol, and the
    random-sign probe within 10 sigma of a tol-sized error (std of sum s_i e_i = ||e||)."""
    got = np.asarray(got, dtype=float).reshape(-1)
    ref_norm = float(z[prefix + "_norm"])
    assert rel_l2(got[::stride], z[prefix + "_sample"]) <= tol
    assert abs(np.linalg.norm(got) - ref_norm) <= tol * ref_norm
    assert abs(got.sum() - float(z[prefix + "_sum"])) <= 10 * tol * ref_norm
    assert abs(got @ _probe(got.size) - float(z[prefix + "_probe"])) <= 10 * tol * ref_norm


@pytest.fixture(scope="module")
def prox128():
    return np.load(GOLD / "bench_prox128.npz")


@pytest.fixture(scope="module")
def config2():
    return config2_inputs(128)


def _config2_problem(inp, dtype, twin=False):
    dev = "cuda"
    u = torch.tensor(inp["u"][:, None], dtype=dtype, device=dev)
    if twin:
        w = W.DiagPlusLowRank(inp["tau_twin"], u)
    else:
        w = W.DiagPlusLowRank(1.0, u, d=torch.tensor(inp["d"], dtype=dtype, device=dev))
    v = torch.tensor(inp["v"], dtype=dtype, device=dev)
    return D.DualTvProblem(grid=bq.Grid((128, 128, 128)), v=v, w=w, reg=inp["reg"], box=W.BoxSet(0.0, np.inf))


def test_config2_headline_fp32_vs_port(prox128, config2):
    """The benched solve itself: 128^3 fp32 diag(d) + u u^T, 100 iterations."""
    rep = D.solve(_config2_problem(config2, torch.float32), eps=1e-300, max_iter=100)
    assert rep.iterations == 100
    check_summary(prox128, "diag_x", rep.x.double().cpu().numpy(), 1e-4)
    check_summary(prox128, "diag_p", rep.p_star.double().cpu().numpy(), 1e-4, stride=3 * STRIDE)
    assert float(rep.x.min()) >= 0.0


def test_config2_fp64_twin_vs_port(prox128, config2):
    rep = D.solve(_config2_problem(config2, torch.float64), eps=1e-300, max_iter=100)
    check_summary(prox128, "diag_x", rep.x.cpu().numpy(), 1e-10)
    check_summary(prox128, "diag_p", rep.p_star.cpu().numpy(), 1e-10, stride=3 * STRIDE)
    assert rep.newton_iterations == int(prox128["diag_newton"])
    assert abs(float(rep.beta_star[0]) - float(prox128["diag_beta"][0])) <= 1e-8 * max(1.0, abs(float(prox128["diag_beta"][0])))


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-10), (torch.float32, 1e-4)])
def test_config2_scalar_tau_twin_vs_reference_solve(prox128, config2, dtype, tol):
    """W = 1.25 I + u u^T at 128^3: the reference's own solve is the fixture."""
    rep = D.solve(_config2_problem(config2, dtype, twin=True), eps=1e-300, max_iter=100)
    check_summary(prox128, "twin_x", rep.x.double().cpu().numpy(), tol)
    check_summary(prox128, "twin_p", rep.p_star.double().cpu().numpy(), tol, stride=3 * STRIDE)
    if dtype == torch.float64:
        assert rep.newton_iterations == int(prox128["twin_newton"])


@pytest.fixture(scope="module")
def ls128():
    z = np.load(GOLD / "bench_ls128.npz")
    vs = PH.ScatterViewSet(128, 64, model="ls", dtype=torch.complex64, theta_deg=40.0, tol=1e-6, max_iter=500,
                           batch=2)
    x = torch.tensor(0.5 * ls_phantom(128, 12, 0.01, 0.1, seed=4000), dtype=torch.float32, device="cuda")
    return z, vs, x


def test_config4_subset_gradient_c64_vs_oracle(ls128):
    z, vs, x = ls128
    views = [int(v) for v in z["views"]]
    vs.y[views] = torch.tensor(z["y"], dtype=torch.float32, device="cuda")
    vs.iters_forward.clear()
    vs.iters_adjoint.clear()
    g = vs.subset_gradient(views, x).double().cpu().numpy()
    check_summary(z, "grad", g, 1e-4)
    # the oracle logs forward then adjoint iterations per view
    ref_it = [int(i) for i in z["grad_iters"]]
    got_it = [vs.iters_forward[0], vs.iters_adjoint[0], vs.iters_forward[1], vs.iters_adjoint[1]]
    assert max(abs(a - b) for a, b in zip(got_it, ref_it)) <= 1


def test_config4_fixed_k_bicgstab_c64_vs_oracle(ls128):
    z, vs, x = ls128
    tol, mi = vs.tol, vs.max_iter
    try:
        vs.tol, vs.max_iter = 0.0, 6
        f, _ = vs.potential(x)
        u, it = vs.solve(False, f, vs.incident([5]))
    finally:
        vs.tol, vs.max_iter = tol, mi
    assert int(it[0]) == 6
    u = u[0].cpu().numpy()
    check_summary(z, "bicg6_re", u.real.astype(float), 1e-4 * np.sqrt(2))
    check_summary(z, "bicg6_im", u.imag.astype(float), 1e-4 * np.sqrt(2))


def test_config3_n64_bqnpm_vs_reference_loop():
    """n = 64 padded to 128^3 runs the pruned line passes inside a pinned
    reconstruction: device loop (c64) vs the reference bqnpm_run on the c128 oracle."""
    z = np.load(GOLD / "bench_config3_64.npz")
    views, vs = PH.make_scatter_views(64, 8, model="ls", dtype=torch.complex64, theta_deg=35.0, batch=4,
                                      tol=1e-6, max_iter=500)
    vs.y.copy_(torch.tensor(z["y"], dtype=torch.float32, device="cuda"))
    grid = bq.Grid((64, 64, 64))
    box = W.BoxSet(0.0, 0.1)
    x0 = S.scaled_adjoint_initializer(views, grid, box)
    assert rel_l2(x0.double().cpu().numpy(), z["x0"]) <= 1e-4
    al = S.estimate_subset_lipschitz(views, S.partition_views(8, 2), torch.tensor(z["x0"], dtype=torch.float32,
                                                                                   device="cuda"), 2, 1.05, 0)
    np.testing.assert_allclose(al, z["alphas"], rtol=1e-4)
    cfg = S.SolverConfig(subsets=2, tv_weight=1e-3, max_outer=3, box=box, seed=0, alphas=z["alphas"])
    xgt = ls_phantom(64, 5, 0.02, 0.08, seed=3000)
    x, tr = S.bqnpm_run(views, grid, cfg, x0=z["x0"], ground_truth=xgt)
    assert rel_l2(x, z["x"]) <= 1e-3
    np.testing.assert_allclose(tr.column("cost"), z["cost"], rtol=1e-3)
    np.testing.assert_allclose(tr.column("snr_db"), z["snr"], atol=0.05)

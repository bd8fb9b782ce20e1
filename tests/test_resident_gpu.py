"""The GPU-resident BQNPM loop (resident.py: device SR1 decisions, compacted
fixed-rank metric, device tau / rank in the prox, CUDA-graph replay) against
the reference golden runs and against the host-decision loop."""

from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_02043_b200 import forward_models as FM  # noqa: E402
from paper_2307_02043_b200 import solvers as S  # noqa: E402
from paper_2307_02043_b200.tv_ops import Grid  # noqa: E402
from paper_2307_02043_b200.wpm import BoxSet  # noqa: E402


def _dct_views(tag, dims):
    g = Grid(dims)
    if tag == "lin":
        return g, FM.make_linear_views(g, 8, mask_fraction=0.5, seed=3, noise_snr_db=30.0)
    return g, FM.make_nonlinear_views(g, 8, strength=0.1, mask_fraction=0.5, seed=3, noise_snr_db=30.0)


@pytest.mark.parametrize("tag,dims", [("lin", (16, 9, 8)), ("nl", (32, 8, 6))])
@pytest.mark.parametrize("graphs", ["1", "0"])
def test_resident_matches_host_loop(monkeypatch, tag, dims, graphs):
    monkeypatch.setenv("BQ_GRAPHS", graphs)
    g, views = _dct_views(tag, dims)
    cfg = S.SolverConfig(subsets=4, tv_weight=2e-3, max_outer=24, box=BoxSet(1.3, 1.4), seed=0)
    xr, tr = S.bqnpm_run(views, g, cfg, resident=True)
    xh, th = S.bqnpm_run(views, g, cfg, resident=False)
    ng = getattr(tr, "graphs", 0)
    assert (ng >= 5) if graphs == "1" else ng == 0  # 4 pre-prox graphs + >= 1 prox graph
    assert rel_l2(xr, xh) <= 1e-11
    np.testing.assert_allclose(tr.column("cost"), th.column("cost"), rtol=1e-11)
    np.testing.assert_array_equal(tr.column("inner_iters"), th.column("inner_iters"))
    np.testing.assert_array_equal(tr.column("grad_evals"), th.column("grad_evals"))


def test_resident_on_iteration_and_snr():
    g, views = _dct_views("lin", (16, 9, 8))
    xgt = FM.make_phantom(g, seed=3).values
    cfg = S.SolverConfig(subsets=4, tv_weight=2e-3, max_outer=12, box=BoxSet(1.3, 1.4), seed=0)
    seen = []
    xr, tr = S.bqnpm_run(views, g, cfg, ground_truth=xgt, resident=True,
                         on_iteration=lambda k, x, row, info: seen.append((k, row.cost)))
    xh, th = S.bqnpm_run(views, g, cfg, ground_truth=xgt, resident=False)
    assert [k for k, _ in seen] == list(range(13))
    np.testing.assert_allclose([c for _, c in seen], th.column("cost"), rtol=1e-11)
    np.testing.assert_allclose(tr.column("snr_db"), th.column("snr_db"), rtol=1e-9)
    assert np.all(np.diff(tr.column("elapsed_s")) >= 0)


def test_resident_born_config1_golden():
    """Config 1 (first Born, c128): the resident loop with graph replay reproduces
    the reference golden run."""
    from paper_2307_02043_b200 import physics as PH

    z = np.load(Path(__file__).parent / "golden" / "config1_golden.npz")
    views, vs = PH.make_scatter_views(32, 16, model="born", dtype=torch.complex128, theta_deg=35.0, batch=8)
    vs.y.copy_(torch.tensor(z["c1_y"], device="cuda"))
    cfg = S.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=20, box=BoxSet(0.0, 0.1), seed=0,
                         alphas=z["c1_alphas"])
    x, tr = S.bqnpm_run(views, Grid((32, 32, 32)), cfg, x0=z["c1_x0"], ground_truth=z["c1_xgt"], resident=True)
    assert tr.graphs >= 5
    assert rel_l2(x, z["c1_x"]) <= 1e-8
    np.testing.assert_allclose(tr.column("cost"), z["c1_cost"], rtol=1e-8)
    np.testing.assert_array_equal(tr.column("inner_iters"), z["c1_inner"])


def test_resident_not_applicable_is_reported():
    from paper_2307_02043_b200 import physics as PH

    views, vs = PH.make_scatter_views(8, 4, model="ls", dtype=torch.complex128, batch=4)
    cfg = S.SolverConfig(subsets=2, tv_weight=1e-3, max_outer=1, box=BoxSet(0.0, 0.1), alphas=[1.0, 1.0])
    with pytest.raises(ValueError):
        S.bqnpm_run(views, Grid((8, 8, 8)), cfg, x0=np.zeros(512), resident=True)

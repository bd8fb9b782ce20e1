"""INTEGRATION.md's drop-in, executed: the UNMODIFIED reference ``bqnpm_run``
(installed under baseline/_ref, which travels to the GPU box) with the
documented names patched to the device implementations, driving device
views, reproduces the reference golden runs (tests/golden/*.npz)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture
def tvqn_patched(monkeypatch):
    if not (REF / "tvqn" / "solvers.py").exists():
        pytest.skip("reference not installed under baseline/_ref (see DESIGN.md, reference arm)")
    monkeypatch.syspath_prepend(str(REF))
    for name in [m for m in sys.modules if m == "tvqn" or m.startswith("tvqn.")]:
        monkeypatch.delitem(sys.modules, name)
    import tvqn.dual_tv_solver as DTS
    import tvqn.solvers as S

    import paper_2307_02043_b200 as bq
    from paper_2307_02043_b200 import dual_tv_solver as bq_dts
    from paper_2307_02043_b200 import forward_models as bq_fm
    from paper_2307_02043_b200 import hessian_sr1 as bq_sr1
    from paper_2307_02043_b200 import metric_ops as bq_m

    # exactly the patch list of INTEGRATION.md section 2
    monkeypatch.setattr(S, "subset_gradient", bq_fm.subset_gradient)
    monkeypatch.setattr(S, "full_cost", bq_fm.full_cost)
    monkeypatch.setattr(S, "estimate_sr1", bq_sr1.estimate_sr1)
    monkeypatch.setattr(S, "aggregate_metric", bq_m.aggregate_metric)
    monkeypatch.setattr(S, "compute_v_k", bq_m.compute_v_k)
    monkeypatch.setattr(S, "DiagPlusLowRank", bq.DiagPlusLowRank)
    monkeypatch.setattr(S, "DualTvProblem", bq_dts.DualTvProblem)
    monkeypatch.setattr(DTS, "solve", bq_dts.solve)
    calls = {"solve": 0}
    orig = bq_dts.solve

    def counting_solve(*a, **k):
        calls["solve"] += 1
        return orig(*a, **k)

    monkeypatch.setattr(DTS, "solve", counting_solve)
    assert S.__file__.startswith(str(REF))
    return S, calls


@pytest.mark.parametrize("tag,strength,dims", [("lin", 0.0, (10, 9, 8)), ("nl", 0.1, (12, 8, 6))])
def test_reference_bqnpm_run_on_device_operators(golden, tvqn_patched, tag, strength, dims):
    S, calls = tvqn_patched
    from paper_2307_02043_b200 import forward_models as FM
    from paper_2307_02043_b200.tv_ops import Grid
    from paper_2307_02043_b200.wpm import BoxSet

    g = Grid(dims)
    if strength == 0.0:
        views = FM.make_linear_views(g, 8, mask_fraction=0.5, seed=3, noise_snr_db=30.0)
    else:
        views = FM.make_nonlinear_views(g, 8, strength=strength, mask_fraction=0.5, seed=3, noise_snr_db=30.0)
    cfg = S.SolverConfig(subsets=4, tv_weight=2e-3, max_outer=10, box=BoxSet(1.3, 1.4), seed=0)
    x, tr = S.bqnpm_run(views, g, cfg)  # the reference's own loop
    assert calls["solve"] == 10
    assert rel_l2(x, golden[f"bqnpm_{tag}_x"]) <= 1e-9
    np.testing.assert_allclose(tr.column("cost"), golden[f"bqnpm_{tag}_cost"], rtol=1e-9)
    np.testing.assert_array_equal(tr.column("inner_iters"), golden[f"bqnpm_{tag}_inner"])


def test_reference_bqnpm_run_on_device_born_views(tvqn_patched):
    """Config 1 (first Born, c128): the reference loop on the device ScatterView
    plugin views reproduces the config-1 golden (made by the same reference loop
    on the CPU Born oracle)."""
    S, calls = tvqn_patched
    from paper_2307_02043_b200 import physics as PH
    from paper_2307_02043_b200.tv_ops import Grid
    from paper_2307_02043_b200.wpm import BoxSet

    z = np.load(Path(__file__).parent / "golden" / "config1_golden.npz")
    views, vs = PH.make_scatter_views(32, 16, model="born", dtype=torch.complex128, theta_deg=35.0, batch=8)
    vs.y.copy_(torch.tensor(z["c1_y"], device="cuda"))
    cfg = S.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=20, box=BoxSet(0.0, 0.1), seed=0,
                         alphas=z["c1_alphas"])
    x, tr = S.bqnpm_run(views, Grid((32, 32, 32)), cfg, x0=z["c1_x0"], ground_truth=z["c1_xgt"])
    assert calls["solve"] == 20
    assert rel_l2(x, z["c1_x"]) <= 1e-8
    np.testing.assert_allclose(tr.column("cost"), z["c1_cost"], rtol=1e-8)

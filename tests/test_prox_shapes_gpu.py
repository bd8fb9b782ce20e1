"""Shape sweep of the fused prox kernel against the general-shape kernel (itself
pinned to the oracle and the reference goldens in test_prox_gpu.py): seeded
random grids over every staged row length, ranks 0-4, diag(d) and scalar tau,
so that the per-tile block assignment, the partial last tile, the x-split rows
and the compact near list meet odd K2 / K3 combinations."""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import dual_tv_solver as D  # noqa: E402
from paper_2307_02043_b200 import wpm as W  # noqa: E402


def _cases():
    rng = np.random.default_rng(20260)
    out = []
    for k1 in (4, 8, 16, 32, 64, 128, 256):
        for _ in range(3):
            k2 = int(rng.integers(3, 60 if k1 <= 64 else 150))
            k3 = int(rng.integers(3, 70 if k1 <= 64 else 40))
            out.append((k1, k2, k3, int(rng.integers(0, 5)), bool(rng.integers(0, 2)), bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("k1,k2,k3,r,diag,f32", _cases())
def test_fused_matches_general_on_random_shapes(monkeypatch, k1, k2, k3, r, diag, f32):
    dims = (k1, k2, k3)
    n = k1 * k2 * k3
    dtype = torch.float32 if f32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(n + r)
    v = torch.randn(n, generator=g, device="cuda", dtype=dtype) * 0.5 + 0.3
    U = torch.randn(n, r, generator=g, device="cuda", dtype=dtype) / np.sqrt(n)
    d = torch.rand(n, generator=g, device="cuda", dtype=dtype) * 1.5 + 0.5 if diag else None
    w = W.DiagPlusLowRank(1.0 if diag else 1.25, U, d=d) if r else (
        W.DiagPlusLowRank(1.0, torch.zeros(n, 0, device="cuda", dtype=dtype), d=d) if diag
        else W.DiagPlusLowRank.diagonal(1.25, n, dtype=dtype))
    prob = D.DualTvProblem(grid=bq.Grid(dims), v=v, w=w, reg=0.05)
    fused = D.solve(prob, eps=1e-300, max_iter=25)
    monkeypatch.setenv("BQ_PROX_GENERAL", "1")
    general = D.solve(prob, eps=1e-300, max_iter=25)
    tol = 1e-4 if f32 else 1e-9
    assert fused.iterations == general.iterations == 25
    assert rel_l2(fused.x.double().cpu().numpy(), general.x.double().cpu().numpy()) <= tol
    assert rel_l2(fused.p_star.double().cpu().numpy(), general.p_star.double().cpu().numpy()) <= tol
    if not f32:
        assert fused.newton_iterations == general.newton_iterations

"""z-slab-sharded prox on the device (csrc/slab_prox.cu through the C ABI): the
sharded solve over several slabs (the loopback layout of one GPU: the halo
planes are device copies, the all-reduces local sums) against the unsharded
device solve and the oracle.  The cross-process path (NCCL send/recv and
all-reduce) is the same control code, checked with gloo in test_slab_prox.py."""

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
from paper_2307_02043_b200 import slab_prox as SP  # noqa: E402
from paper_2307_02043_b200 import wpm as W  # noqa: E402


@pytest.mark.parametrize("dims,r,diag,iso,nslab", [((24, 20, 16), 1, True, True, 4), ((16, 12, 30), 2, False, False, 3),
                                                   ((20, 18, 9), 0, False, True, 9), ((32, 32, 32), 4, False, True, 8),
                                                   # K1 % 4 != 0: the one-voxel-per-thread passes
                                                   ((18, 10, 12), 1, True, True, 3), ((22, 9, 8), 2, False, False, 4)])
def test_sharded_matches_unsharded_f64(dims, r, diag, iso, nslab):
    rng = np.random.default_rng(r + 10)
    n = int(np.prod(dims))
    v = rng.standard_normal(n) * 0.5 + 0.3
    U = rng.standard_normal((n, r)) / np.sqrt(n)
    d = rng.uniform(0.5, 2.0, n) if diag else None
    w = W.DiagPlusLowRank(1.0 if diag else 1.25, U, d=d) if r else W.DiagPlusLowRank.diagonal(1.25, n)
    box = W.BoxSet(0.0, np.inf) if iso else W.BoxSet(0.0, 1.0)
    mode = "iso" if iso else "aniso"
    single = D.solve(D.DualTvProblem(grid=bq.Grid(dims), v=v, w=w, reg=0.05, mode=mode, box=box), eps=1e-300,
                     max_iter=40)
    rep, mine = SP.solve_sharded(bq.Grid(dims), v, w, 0.05, box, slabs_per_rank=nslab, mode=mode, eps=1e-300,
                                 max_iter=40)
    assert len(mine) == nslab
    assert rel_l2(rep.x.cpu().numpy(), single.x) <= 1e-10
    assert rel_l2(rep.p_star.cpu().numpy(), single.p_star) <= 1e-10
    assert rep.iterations == single.iterations == 40
    assert rep.newton_iterations == single.newton_iterations
    ref = O.fgp_prox(dims, v, O.Metric(tau=None if diag else (1.0 if diag else 1.25), U=U if r else None,
                                       d=d, n=n), reg=0.05, hi=np.inf if iso else 1.0, isotropic=iso,
                     eps=1e-300, max_iter=40)
    assert rel_l2(rep.x.cpu().numpy(), ref["x"]) <= 1e-10


def test_sharded_config2_law_f32_and_converged_stop():
    """fp32, the config-2 law at 64^3 over 8 slabs (the config-5 split of 256 planes
    over 8 ranks, scaled), and a tolerance-stopped solve (eps 1e-4)."""
    from paper_2307_02043_b200.configs import config2_inputs

    inp = config2_inputs(64)
    dev = "cuda"
    w = W.DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=torch.float32, device=dev),
                          d=torch.tensor(inp["d"], dtype=torch.float32, device=dev))
    v = torch.tensor(inp["v"], dtype=torch.float32, device=dev)
    g = bq.Grid((64, 64, 64))
    ref = O.fgp_prox((64, 64, 64), inp["v"], O.Metric(U=inp["u"][:, None], d=inp["d"]), reg=0.05, eps=1e-300,
                     max_iter=100)
    rep, _ = SP.solve_sharded(g, v, w, 0.05, W.BoxSet(0.0, np.inf), slabs_per_rank=8, eps=1e-300, max_iter=100)
    assert rel_l2(rep.x.double().cpu().numpy(), ref["x"]) <= 1e-4
    single = D.solve(D.DualTvProblem(grid=g, v=v, w=w, reg=0.05), eps=1e-4, max_iter=500)
    rep2, _ = SP.solve_sharded(g, v, w, 0.05, W.BoxSet(0.0, np.inf), slabs_per_rank=8, eps=1e-4, max_iter=500)
    assert rep2.converged and single.converged
    assert abs(rep2.iterations - single.iterations) <= 1
    assert rel_l2(rep2.x.double().cpu().numpy(), single.x.double().cpu().numpy()) <= 1e-4

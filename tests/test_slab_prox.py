"""z-slab-sharded prox: the control code of paper_2307_02043_b200/slab_prox.py
(halo exchange, all-reduces, replicated Newton and FGP decisions) with the
numpy pass backend (oracle/slab.py), in one process over several slabs and
over gloo at world size 2, against the unsharded oracle prox
(oracle/prox.py, which follows dual_tv_solver.py:161-250)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import prox as O
from oracle.slab import NumpySlabs
from paper_2307_02043_b200 import slab_prox as SP


def _case(kind):
    rng = np.random.default_rng({"diag": 1, "tau2": 2, "rank0": 3, "neg": 4}[kind])
    dims = (9, 7, 11)
    n = int(np.prod(dims))
    v = rng.standard_normal(n) * 0.5 + 0.3
    if kind == "diag":
        d = rng.uniform(0.5, 2.0, n)
        U = rng.standard_normal((n, 1)) / np.sqrt(n)
        return dims, v, dict(U=U, d=d, tau=1.0, sign=1, lo=0.0, hi=np.inf, iso=True, reg=0.05)
    if kind == "tau2":
        U = rng.standard_normal((n, 2)) / np.sqrt(n)
        return dims, v, dict(U=U, d=None, tau=1.3, sign=1, lo=0.0, hi=1.0, iso=False, reg=0.08)
    if kind == "neg":
        U = rng.standard_normal((n, 2)) * 0.5 / np.sqrt(n)
        return dims, v, dict(U=U, d=None, tau=1.3, sign=-1, lo=-0.2, hi=0.9, iso=True, reg=0.05)
    return dims, v, dict(U=np.zeros((n, 0)), d=None, tau=0.9, sign=1, lo=0.0, hi=np.inf, iso=True, reg=0.05)


def _oracle(dims, v, c, max_iter):
    w = O.Metric(tau=c["tau"] if c["d"] is None else None, U=c["U"], sign=c["sign"], d=c["d"], n=v.size)
    return O.fgp_prox(dims, v, w, reg=c["reg"], lo=c["lo"], hi=c["hi"], isotropic=c["iso"], eps=1e-300,
                      max_iter=max_iter)


def _slab_run(dims, v, c, bounds, comm, max_iter):
    r = c["U"].shape[1]
    be = NumpySlabs(dims, bounds, dims[2], v, c["U"], c["d"], rank=r, sign=c["sign"], tau=c["tau"], reg=c["reg"],
                    lo=c["lo"], hi=c["hi"], iso=c["iso"])
    w = O.Metric(tau=c["tau"] if c["d"] is None else None, U=c["U"], sign=c["sign"], d=c["d"], n=v.size)
    gram = (c["U"].T @ (c["U"] / c["d"][:, None]) if c["d"] is not None else c["U"].T @ c["U"]) if r else None
    omega = 1.0 / w.min_diag()
    step = 1.0 / (4.0 * 3 * omega * c["reg"])
    sg = SP.SlabGroup(be, comm, dims, bounds, dims[2])
    return SP.slab_solve(sg, rank=r, sign=c["sign"], tau=c["tau"], scalar=c["d"] is None, gram=gram,
                         reg=c["reg"], step=step, eps=1e-300, max_iter=max_iter)


def test_slab_bounds_partition():
    for k3 in (1, 5, 32, 256):
        for w in (1, 2, 3, 8):
            if w > k3:
                continue
            b = SP.slab_bounds(k3, w)
            assert b[0][0] == 0 and b[-1][1] == k3
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            sizes = [z1 - z0 for z0, z1 in b]
            assert max(sizes) - min(sizes) <= 1
    assert SP.slab_bounds(256, 8) == [(32 * i, 32 * (i + 1)) for i in range(8)]  # config 5


@pytest.mark.parametrize("kind", ["diag", "tau2", "rank0", "neg"])
@pytest.mark.parametrize("nslab", [1, 3, 11])
def test_loopback_slabs_match_unsharded_oracle(kind, nslab):
    dims, v, c = _case(kind)
    ref = _oracle(dims, v, c, 25)
    rep = _slab_run(dims, v, c, SP.slab_bounds(dims[2], nslab), SP.Comm(None), 25)
    assert np.linalg.norm(rep.x.numpy() - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])
    assert np.linalg.norm(rep.p_star.numpy() - ref["p_star"]) <= 1e-12 * np.linalg.norm(ref["p_star"])
    assert rep.iterations == ref["iterations"]
    assert rep.newton_iterations == ref["newton_iterations"]
    if c["U"].shape[1]:
        np.testing.assert_allclose(rep.beta_star, ref["beta_star"], rtol=1e-9, atol=1e-12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, per_rank, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, v, c = _case(kind)
        allb = SP.slab_bounds(dims[2], world * per_rank)
        mine = allb[rank * per_rank:(rank + 1) * per_rank]
        rep = _slab_run(dims, v, c, mine, SP.Comm(None), 25)
        out[rank] = (rep.x.numpy(), rep.p_star.numpy(), rep.iterations, rep.newton_iterations, rep.beta_star)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,per_rank", [("diag", 1), ("tau2", 2), ("neg", 1)])
def test_gloo_world2_slab_prox_matches_unsharded(kind, per_rank):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, kind, per_rank, out), nprocs=2, join=True)
    dims, v, c = _case(kind)
    ref = _oracle(dims, v, c, 25)
    x = np.concatenate([out[0][0], out[1][0]])
    p = np.concatenate([out[0][1], out[1][1]], axis=1)
    assert np.linalg.norm(x - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])
    assert np.linalg.norm(p - ref["p_star"]) <= 1e-12 * np.linalg.norm(ref["p_star"])
    for r in range(2):
        assert out[r][2] == ref["iterations"] and out[r][3] == ref["newton_iterations"]
    np.testing.assert_array_equal(out[0][4], out[1][4])  # replicated controller: identical beta on both ranks


@pytest.mark.parametrize("kind", ["diag", "tau2"])
def test_tolerance_stop_undoes_the_speculative_iteration(kind):
    """eps-stopped solve: the next iteration is queued before the stop test is
    known and must be undone (beta, Newton count) -- same result as the oracle."""
    dims, v, c = _case(kind)
    w = O.Metric(tau=c["tau"] if c["d"] is None else None, U=c["U"], sign=c["sign"], d=c["d"], n=v.size)
    ref = O.fgp_prox(dims, v, w, reg=c["reg"], lo=c["lo"], hi=c["hi"], isotropic=c["iso"], eps=2e-3, max_iter=500)
    r = c["U"].shape[1]
    be = NumpySlabs(dims, SP.slab_bounds(dims[2], 3), dims[2], v, c["U"], c["d"], rank=r, sign=c["sign"],
                    tau=c["tau"], reg=c["reg"], lo=c["lo"], hi=c["hi"], iso=c["iso"])
    gram = (c["U"].T @ (c["U"] / c["d"][:, None]) if c["d"] is not None else c["U"].T @ c["U"]) if r else None
    step = 1.0 / (4.0 * 3 * (1.0 / w.min_diag()) * c["reg"])
    sg = SP.SlabGroup(be, SP.Comm(None), dims, SP.slab_bounds(dims[2], 3), dims[2])
    rep = SP.slab_solve(sg, rank=r, sign=c["sign"], tau=c["tau"], scalar=c["d"] is None, gram=gram, reg=c["reg"],
                        step=step, eps=2e-3, max_iter=500)
    assert ref["converged"] and rep.converged and rep.iterations == ref["iterations"] < 500
    assert rep.newton_iterations == ref["newton_iterations"]
    assert rep.rel_change == pytest.approx(ref["rel_change"], rel=1e-9)
    assert np.linalg.norm(rep.x.numpy() - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])

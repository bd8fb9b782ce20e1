"""Multi-process (gloo, world size 2, CPU) tests of the view-sharded subset
gradient: the host logic that runs over NCCL on GPUs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_02043_b200 import dist as D


def test_shard_is_contiguous_balanced_partition():
    for n in range(0, 40):
        for w in (1, 2, 3, 4, 8):
            idx = list(range(100, 100 + n))
            parts = [D.shard(idx, r, w) for r in range(w)]
            assert sum(parts, []) == idx
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    # config 5: 30-view subsets over 8 GPUs -> 4/4/4/4/4/4/3/3
    assert [len(D.shard(range(30), r, 8)) for r in range(8)] == [4, 4, 4, 4, 4, 4, 3, 3]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _CpuViews:
    """Stand-in view set with the device API (subset_gradient(chunk, x)), backed by
    the numpy oracle of the reference's masked-spectrum views."""

    def __init__(self):
        from oracle import views as OV
        from paper_2307_02043_b200.forward_models import spectrum_masks
        from paper_2307_02043_b200.tv_ops import Grid

        self.dims = (8, 7, 6)
        rng = np.random.default_rng(0)
        masks, _ = spectrum_masks(Grid(self.dims), 6, 0.5)
        n = int(np.prod(self.dims))
        self.views = [OV.DctView(self.dims, masks[i], rng.standard_normal(n) * masks[i], 0.1) for i in range(6)]

    def subset_gradient(self, chunk, x):
        from oracle import views as OV

        return torch.from_numpy(OV.subset_gradient(self.views, chunk, x.numpy()))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vs = _CpuViews()
        x = torch.from_numpy(np.random.default_rng(1).standard_normal(int(np.prod(vs.dims))))
        g = D.subset_gradient(vs, [0, 2, 3, 5, 1], x)
        out[rank] = g.numpy()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_single_process():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    vs = _CpuViews()
    from oracle import views as OV

    x = np.random.default_rng(1).standard_normal(int(np.prod(vs.dims)))
    ref = OV.subset_gradient(vs.views, [0, 2, 3, 5, 1], x)
    for r in range(2):
        np.testing.assert_allclose(out[r], ref, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(out[0], out[1])  # replicas agree bit for bit

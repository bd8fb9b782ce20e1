"""View-sharded multi-GPU execution.

One process per GPU (torchrun).  For subset S_t (``partition_views``,
solvers.py:41-55) rank g takes a contiguous chunk of S_t's index list (chunk
sizes differ by <= 1), sums its views' gradients in fixed order on its GPU,
and ONE all-reduce (NCCL over NVLink; gloo in the CPU tests) of the N-vector
gives sum_{rho in S_t} grad f_rho on every rank; dividing by |S_t| gives the
reference's ``subset_gradient`` (forward_models.py:304-309).  Everything else
(SR1, aggregate metric, v_k, prox) is replicated: the kernels are
deterministic, so all ranks hold bit-identical iterates without a broadcast.
Changing the rank count changes only the floating-point summation order.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard(indices, rank, world):
    """Contiguous chunk of `indices` for `rank` (sizes differ by <= 1)."""
    idx = list(indices)
    n = len(idx)
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return idx[start:start + size]


def world_info(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_sum(partial_sum, indices, like: torch.Tensor, group=None):
    """sum over `indices` of per-view terms: partial_sum(chunk) on each rank
    (returns an unnormalised N-vector, or None for an empty chunk), then one
    all-reduce(SUM)."""
    rank, world = world_info(group)
    chunk = shard(indices, rank, world)
    acc = partial_sum(chunk) if chunk else None
    if acc is None:
        acc = torch.zeros_like(like)
    if world > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def subset_gradient(viewset, view_ids, x, group=None):
    """Distributed ``subset_gradient`` for a device view set (DctViewSet or
    ScatterViewSet): each rank evaluates its chunk, one all-reduce, / |S|."""
    ids = list(view_ids)

    def part(chunk):
        return viewset.subset_gradient(chunk, x) * float(len(chunk))

    g = sharded_sum(part, ids, x, group)
    return g / float(len(ids))


__all__ = ["shard", "world_info", "sharded_sum", "subset_gradient"]

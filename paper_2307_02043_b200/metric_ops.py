"""Slot aggregation and the metric-weighted centre v_k on the device.

Mirrors ``tvqn.solvers`` (``/root/reference/pkg/src/tvqn/solvers.py``):
``kappa`` (:29-38), ``partition_views`` (:41-55), ``SubsetSlot`` (:58-64),
``aggregate_metric`` (:67-77) and ``compute_v_k`` (:80-89).  v_k runs in
``bq_vk``: u_t^T x_t dots, the slot sum and the Woodbury inverse with the
capacitance factorised on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._tensors import default_device, is_torch, out_like, pick_dtype, to_dev
from .hessian_sr1 import Sr1Estimate
from .wpm import DiagPlusLowRank


def kappa(k, t, n_subsets):
    if not 1 <= t <= n_subsets:
        raise ValueError(f"term index {t} out of range [1, {n_subsets}]")
    return (k - 1 - t) % n_subsets + 1


def partition_views(n_views, n_subsets, strategy="equispaced"):
    if not 1 <= n_subsets <= n_views:
        raise ValueError(f"need 1 <= n_subsets <= {n_views}, got {n_subsets}")
    idx = np.arange(n_views)
    if strategy == "equispaced":
        return [idx[t::n_subsets] for t in range(n_subsets)]
    if strategy == "contiguous":
        return list(np.array_split(idx, n_subsets))
    raise ValueError(f"unknown partition strategy: {strategy!r}")


@dataclass
class SubsetSlot:
    x: object
    grad: object
    hess: Sr1Estimate


def aggregate_metric(slots, dtype=None) -> DiagPlusLowRank:
    """tau = sum tau_t, columns = nonzero u_t in slot order, sign + (solvers.py:67-77)."""
    tau = sum(s.hess.tau for s in slots)
    cols = [s.hess.u for s in slots if s.hess.u is not None]
    x0 = slots[0].x
    dtype = dtype or pick_dtype(x0)
    dev = x0.device if is_torch(x0) and x0.is_cuda else default_device()
    n = x0.shape[0]
    if cols:
        U = torch.stack([to_dev(c, dtype, dev) for c in cols], dim=1)
    else:
        U = torch.zeros(n, 0, dtype=dtype, device=dev)
    return DiagPlusLowRank(tau=tau, U=U, dtype=dtype, device=dev)


def compute_v_k(slots, w: DiagPlusLowRank, step):
    """v = W^-1 sum_t (tau_t x_t + u_t (u_t^T x_t) - step g_t) (solvers.py:80-89)."""
    if len(slots) > 8:
        raise ValueError("at most 8 slots (BQ_MAX_RANK)")
    if w.d is not None:
        # the reference's aggregated metric is tau I + U U^T (solvers.py:67-77); bq_vk has no d
        raise ValueError("compute_v_k needs a scalar-tau metric (aggregate_metric), not a per-voxel diagonal")
    dtype, dev = w.dtype, w.device
    xs = [to_dev(s.x, dtype, dev) for s in slots]
    gs = [to_dev(s.grad, dtype, dev) for s in slots]
    us = [None if s.hess.u is None else to_dev(s.hess.u, dtype, dev) for s in slots]
    taus = (C.c_double * len(slots))(*[float(s.hess.tau) for s in slots])
    n = xs[0].numel()
    acc = torch.empty(n, dtype=dtype, device=dev)
    out = torch.empty(n, dtype=dtype, device=dev)
    lib = _abi.load_library()
    _abi.check(
        lib.bq_vk(_abi.ctx_for(dev), _abi.dtype_code(dtype), n, len(slots), _abi.ptr_array(xs), _abi.ptr_array(gs),
                  _abi.ptr_array(us), taus, float(step), w.rank, w.sign, w.tau if w.d is None else 0.0,
                  _abi.ptr(w.Ut) if w.rank else None, _abi.ptr(w.gram), acc.data_ptr(), out.data_ptr(),
                  _abi.stream_ptr(dev)),
        "compute_v_k",
    )
    return out_like(slots[0].x, out)


__all__ = ["kappa", "partition_views", "SubsetSlot", "aggregate_metric", "compute_v_k"]

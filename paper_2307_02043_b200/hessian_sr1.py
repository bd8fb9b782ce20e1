"""Memory-frugal SR1 curvature estimate on the device.

Mirror of ``tvqn.hessian_sr1`` (``/root/reference/pkg/src/tvqn/hessian_sr1.py``):
``Sr1Estimate`` (:21-49) and ``estimate_sr1(s, m, gamma, alpha_fallback)``
(:52-101).  The three dot-product passes and every branch of the skip rule run
in ``bq_sr1`` (fixed-order device reductions); the scalars stay on the device
for GPU-resident callers (``estimate_sr1_async``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._tensors import default_device, is_torch, out_like, pick_dtype, to_dev


@dataclass(frozen=True, eq=False)
class Sr1Estimate:
    """B = tau*I + u u^T (u None for rank 0)."""

    tau: float
    u: object = None

    def __post_init__(self):
        if not self.tau > 0:
            raise ValueError(f"tau must be positive, got {self.tau}")
        if self.u is not None:
            zero = (not bool(torch.any(self.u != 0))) if is_torch(self.u) else (not np.any(self.u))
            if zero:
                object.__setattr__(self, "u", None)

    @property
    def rank(self):
        return 0 if self.u is None else 1

    def apply(self, x):
        if is_torch(x) or is_torch(self.u):
            xt = x if is_torch(x) else torch.as_tensor(x)
            out = self.tau * xt
            if self.u is not None:
                out = out + self.u * torch.dot(self.u, xt)
            return out
        out = self.tau * np.asarray(x, dtype=float)
        if self.u is not None:
            out = out + self.u * float(np.dot(self.u, x))
        return out

    def dense(self, n):
        b = self.tau * np.eye(n)
        if self.u is not None:
            u = self.u.detach().cpu().numpy() if is_torch(self.u) else self.u
            b += np.outer(u, u)
        return b


class Sr1Device:
    """Device result of one estimate: est = [tau, has_u, sm, curv, mm, nnz, |s|, |r|, status]."""

    def __init__(self, est: torch.Tensor, u: torch.Tensor):
        self.est = est
        self.u = u


def estimate_sr1_async(s: torch.Tensor, m: torch.Tensor, gamma=0.8, alpha_fallback=1.0) -> Sr1Device:
    if not 0.0 < gamma < 1.0:
        raise ValueError(f"gamma must lie in (0, 1), got {gamma}")
    if not alpha_fallback > 0:
        raise ValueError(f"alpha_fallback must be positive, got {alpha_fallback}")
    if s.shape != m.shape:
        raise ValueError("s and m must have the same shape")
    u = torch.empty_like(s)
    est = torch.zeros(16, dtype=torch.float64, device=s.device)
    lib = _abi.load_library()
    _abi.check(
        lib.bq_sr1(_abi.ctx_for(s.device), _abi.dtype_code(s.dtype), s.numel(), s.data_ptr(), m.data_ptr(),
                   float(gamma), float(alpha_fallback), u.data_ptr(), est.data_ptr(), _abi.stream_ptr(s.device)),
        "estimate_sr1",
    )
    return Sr1Device(est, u)


def estimate_sr1(s, m, gamma=0.8, alpha_fallback=1.0) -> Sr1Estimate:
    """Drop-in for ``tvqn.hessian_sr1.estimate_sr1`` (hessian_sr1.py:52-101)."""
    dtype = pick_dtype(s, m)
    dev = s.device if is_torch(s) and s.is_cuda else default_device()
    st = to_dev(s, dtype, dev)
    mt = to_dev(m, dtype, dev)
    r = estimate_sr1_async(st, mt, gamma, alpha_fallback)
    e = r.est.cpu().numpy()
    if e[8] != 0.0:
        raise ValueError("degenerate step: s must be nonzero")
    tau = float(e[0])
    if e[1] > 0:
        return Sr1Estimate(tau=tau, u=out_like(s, r.u))
    return Sr1Estimate(tau=tau)


__all__ = ["Sr1Estimate", "estimate_sr1", "estimate_sr1_async", "Sr1Device"]

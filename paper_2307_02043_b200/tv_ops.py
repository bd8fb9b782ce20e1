"""Grid / TV-mode descriptors and the device TV value.

Mirrors the public surface of the reference ``tvqn.tv_ops`` that the hot
path touches (``/root/reference/pkg/src/tvqn/tv_ops.py``):

* ``Grid`` (:42-99): dims, size, Fortran strides, ndim.  Flat order is
  Fortran over ``dims`` (dims[0] fastest) == a C-order torch tensor of shape
  ``dims[::-1]``; every device kernel uses that layout.
* ``TvMode`` (:19-39) with the same aliases.
* ``tv_value`` (:162-167) runs on the device (``bq_tv_value``).
* ``apply_diff`` / ``apply_diff_adjoint`` (:107-133), ``gradient_stack`` /
  ``dual_adjoint`` (:136-148), ``dual_divergence`` (:151-159),
  ``project_dual`` (:170-180) and ``diff_operator_norm_sq`` (:183-203) run the
  standalone stencil kernels of ``csrc/tv_stencil.cu``.  Inside the prox the
  same stencils are fused into the persistent kernel and never launched alone;
  these serve the reference's public helpers (``w_of_p``, ``dual_gradient``,
  the objectives).
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from ._tensors import is_torch, out_like, pick_dtype, to_dev


class TvMode(enum.Enum):
    ISOTROPIC = "isotropic"
    ANISOTROPIC = "anisotropic"

    @classmethod
    def parse(cls, value):
        if isinstance(value, TvMode):
            return value
        if isinstance(value, enum.Enum):  # e.g. the reference's own tvqn.tv_ops.TvMode (drop-in)
            value = value.value
        table = {
            "iso": cls.ISOTROPIC,
            "isotropic": cls.ISOTROPIC,
            "aniso": cls.ANISOTROPIC,
            "anisotropic": cls.ANISOTROPIC,
            "l1": cls.ANISOTROPIC,
        }
        try:
            return table[str(value).strip().lower()]
        except KeyError:
            raise ValueError(f"unknown TV mode: {value!r}") from None

    @property
    def code(self) -> int:
        return _abi.BQ_TV_ISO if self is TvMode.ISOTROPIC else _abi.BQ_TV_ANISO


@dataclass(frozen=True)
class Grid:
    """Image geometry: side lengths (K_1, ..., K_d), d in {1, 2, 3}."""

    dims: tuple
    size: int = field(init=False)
    strides: tuple = field(init=False)

    def __post_init__(self):
        dims = tuple(int(k) for k in self.dims)
        if len(dims) not in (1, 2, 3):
            raise ValueError(f"grid must be 1-, 2- or 3-dimensional, got {dims}")
        if min(dims) < 1:
            raise ValueError(f"grid side lengths must be positive, got {dims}")
        strides = tuple(int(np.prod(dims[:i])) for i in range(len(dims)))
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "size", int(np.prod(dims)))
        object.__setattr__(self, "strides", strides)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def dims3(self) -> tuple:
        """dims padded with ones to three entries (the kernels' K1, K2, K3)."""
        return self.dims + (1,) * (3 - len(self.dims))

    def to_nd(self, x):
        a = np.asarray(x)
        if a.size != self.size:
            raise ValueError(f"expected {self.size} entries, got {a.size}")
        return a.reshape(self.dims, order="F")

    def from_nd(self, a):
        a = np.asarray(a)
        if a.shape != self.dims:
            raise ValueError(f"expected shape {self.dims}, got {a.shape}")
        return a.reshape(-1, order="F")


def tv_value(grid: Grid, x, mode=TvMode.ISOTROPIC) -> float:
    """Isotropic / anisotropic TV of ``x`` on the device (``bq_tv_value``)."""
    t = tv_value_async(grid, x, mode)
    return float(t.item())


def tv_value_async(grid: Grid, x, mode=TvMode.ISOTROPIC) -> torch.Tensor:
    """Device scalar (float64 tensor) holding TV(x); no host sync."""
    dt = pick_dtype(x)
    xt = to_dev(x, dt)
    if xt.numel() != grid.size:
        raise ValueError(f"expected {grid.size} entries, got {xt.numel()}")
    out = torch.empty(1, dtype=torch.float64, device=xt.device)
    dims = (C.c_int64 * 3)(*grid.dims3)
    lib = _abi.load_library()
    _abi.check(
        lib.bq_tv_value(
            _abi.ctx_for(xt.device), _abi.dtype_code(dt), grid.ndim, dims, TvMode.parse(mode).code,
            xt.data_ptr(), out.data_ptr(), _abi.stream_ptr(xt.device),
        ),
        "tv_value",
    )
    return out


def _dims_arg(grid: Grid):
    return (C.c_int64 * 3)(*grid.dims3)


def _check_dim(grid: Grid, n):
    if not 1 <= n <= grid.ndim:
        raise ValueError(f"dimension index {n} out of range for {grid.ndim}-D grid")


def _field(grid: Grid, x):
    dt = pick_dtype(x)
    xt = to_dev(x, dt)
    if xt.numel() != grid.size:
        raise ValueError(f"expected {grid.size} entries, got {xt.numel()}")
    return dt, xt.reshape(-1)


def _diff(grid, x, n, adjoint):
    _check_dim(grid, n)
    dt, xt = _field(grid, x)
    out = torch.empty_like(xt)
    lib = _abi.load_library()
    _abi.check(lib.bq_tv_diff(_abi.ctx_for(xt.device), _abi.dtype_code(dt), grid.ndim, _dims_arg(grid), int(n),
                              int(adjoint), xt.data_ptr(), out.data_ptr(), _abi.stream_ptr(xt.device)),
               "apply_diff_adjoint" if adjoint else "apply_diff")
    return out_like(x, out)


def apply_diff(grid: Grid, x, n):
    """Forward difference along dimension n (1-based), zero on the far face (tv_ops.py:107-119)."""
    return _diff(grid, x, n, False)


def apply_diff_adjoint(grid: Grid, y, n):
    """Exact adjoint of ``apply_diff`` along dimension n (tv_ops.py:122-133)."""
    return _diff(grid, y, n, True)


def gradient_stack(grid: Grid, x):
    """[D^1 x; ...; D^d x], shape (d, N) (tv_ops.py:136-143)."""
    dt, xt = _field(grid, x)
    out = torch.empty(grid.ndim, grid.size, dtype=dt, device=xt.device)
    lib = _abi.load_library()
    _abi.check(lib.bq_tv_grad_stack(_abi.ctx_for(xt.device), _abi.dtype_code(dt), grid.ndim, _dims_arg(grid),
                                    xt.data_ptr(), out.data_ptr(), _abi.stream_ptr(xt.device)), "gradient_stack")
    return out_like(x, out)


dual_adjoint = gradient_stack  # tv_ops.py:146-148


def dual_divergence(grid: Grid, p):
    """sum_n (D^n)^T p_n (tv_ops.py:151-159)."""
    shape = tuple(p.shape) if is_torch(p) else np.shape(p)
    if shape != (grid.ndim, grid.size):
        raise ValueError(f"dual field must have shape {(grid.ndim, grid.size)}, got {shape}")
    dt = pick_dtype(p)
    pt = to_dev(p, dt)
    out = torch.empty(grid.size, dtype=dt, device=pt.device)
    lib = _abi.load_library()
    _abi.check(lib.bq_tv_divergence(_abi.ctx_for(pt.device), _abi.dtype_code(dt), grid.ndim, _dims_arg(grid),
                                    pt.data_ptr(), out.data_ptr(), _abi.stream_ptr(pt.device)), "dual_divergence")
    return out_like(p, out)


def project_dual(p, mode=TvMode.ISOTROPIC):
    """Per-voxel projection onto the TV dual set: unit l2 ball (iso) or [-1, 1] (aniso)
    (tv_ops.py:170-180)."""
    dt = pick_dtype(p)
    pt = to_dev(p, dt)
    if pt.ndim == 1:
        pt = pt.reshape(1, -1)
    d, n = pt.shape
    out = torch.empty_like(pt)
    lib = _abi.load_library()
    _abi.check(lib.bq_tv_project_dual(_abi.ctx_for(pt.device), _abi.dtype_code(dt), d, n, TvMode.parse(mode).code,
                                      pt.data_ptr(), out.data_ptr(), _abi.stream_ptr(pt.device)), "project_dual")
    out = out.reshape(p.shape) if is_torch(p) else out.reshape(np.shape(p))
    return out_like(p, out)


def diff_operator_norm_sq(grid: Grid, iters=200, seed=0):
    """Largest eigenvalue of sum_n (D^n)^T D^n by power iteration (tv_ops.py:183-203),
    every product on the device."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(grid.size)
    v /= np.linalg.norm(v)
    vt = to_dev(v, torch.float64)
    lam = 0.0
    for _ in range(iters):
        w = dual_divergence(grid, gradient_stack(grid, vt))
        lam = float(torch.dot(vt, w).item())
        nw = float(torch.linalg.vector_norm(w).item())
        if nw == 0.0:
            return 0.0
        vt = w / nw
    return lam


def power_upper_bound(grid: Grid):
    """Analytic bound 4d on ``diff_operator_norm_sq`` (tv_ops.py:204-206)."""
    return 4.0 * grid.ndim


def tv_maximizing_field(grid: Grid, x, mode=TvMode.ISOTROPIC):
    """Dual field attaining TV(x) in the duality pairing; zero-gradient columns stay 0
    (tv_ops.py:209-220)."""
    g = gradient_stack(grid, x if is_torch(x) else to_dev(x, torch.float64))
    if TvMode.parse(mode) is TvMode.ISOTROPIC:
        norms = torch.sqrt(torch.sum(g * g, dim=0))
        out = g / torch.where(norms > 0, norms, torch.ones_like(norms))
    else:
        out = torch.sign(g)
    return out_like(x, out)


def dual_pairing(grid: Grid, p, x):
    """<d(P), x> (tv_ops.py:223-225)."""
    dv = dual_divergence(grid, p if is_torch(p) else to_dev(p, torch.float64))
    xt = to_dev(x, dv.dtype, dv.device).reshape(-1)
    return float(torch.dot(dv, xt).item())


__all__ = ["Grid", "TvMode", "tv_value", "tv_value_async", "apply_diff", "apply_diff_adjoint", "gradient_stack",
           "dual_adjoint", "dual_divergence", "project_dual", "diff_operator_norm_sq", "power_upper_bound",
           "tv_maximizing_field", "dual_pairing"]

"""Grid / TV-mode descriptors and the device TV value.

Mirrors the public surface of the reference ``tvqn.tv_ops`` that the hot
path touches (``/root/reference/pkg/src/tvqn/tv_ops.py``):

* ``Grid`` (:42-99): dims, size, Fortran strides, ndim.  Flat order is
  Fortran over ``dims`` (dims[0] fastest) == a C-order torch tensor of shape
  ``dims[::-1]``; every device kernel uses that layout.
* ``TvMode`` (:19-39) with the same aliases.
* ``tv_value`` (:162-167) runs on the device (``bq_tv_value``).

The difference stencils and the dual projection themselves are fused into
the prox kernel (``csrc/wtv_prox.cu``); they are not exposed as separate
launches because the hot path never calls them alone.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from ._tensors import to_dev, pick_dtype


class TvMode(enum.Enum):
    ISOTROPIC = "isotropic"
    ANISOTROPIC = "anisotropic"

    @classmethod
    def parse(cls, value):
        if isinstance(value, TvMode):
            return value
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


__all__ = ["Grid", "TvMode", "tv_value", "tv_value_async"]

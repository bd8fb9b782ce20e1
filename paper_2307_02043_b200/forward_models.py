"""Masked-spectrum multi-view measurement models on the device.

Mirror of ``tvqn.forward_models`` (``/root/reference/pkg/src/tvqn/forward_models.py``):

* ``ViewProblem`` (:25-83): forward / jacobian_vec / adjoint_vec / value /
  gradient / self_check with the reference's semantics (numpy in, numpy out).
* ``spectrum_masks`` (:94-136), ``make_phantom`` (:242-282), ``snr_db``
  (:219-228): host-side input construction, re-exported from ``fixtures``
  (restated laws, same RNG use).
* ``make_linear_views`` / ``make_nonlinear_views`` (:153-215): the views of
  one call form a ``DctViewSet`` whose operators run in libbq (exact
  orthonormal DCT per axis, 3-point smoother, pointwise chain rule); the
  construction consumes the seeded RNG exactly like the reference (noise per
  view, then the ``self_check`` draws), so the measurements agree with the
  reference's to rounding.
* ``subset_gradient`` (:304-309), ``subset_value``, ``data_fidelity``,
  ``full_cost`` (:286-301): when the views share one ``DctViewSet`` the whole
  subset is ONE forward DCT + ONE fused mask-combine + ONE inverse DCT.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._tensors import default_device, is_torch, out_like, to_dev
from .tv_ops import Grid, TvMode, tv_value

# host-side input construction (restated reference laws, not the hot path)
from .fixtures import Phantom, make_phantom, snr_db, spectrum_masks  # noqa: E402,F401


# ---------------------------------------------------------------------------
# device view set
# ---------------------------------------------------------------------------
class DctViewSet:
    """L masked-spectrum views of one grid, resident on the device."""

    def __init__(self, grid: Grid, masks, strength=0.0, dtype=torch.float64, device=None):
        if strength < 0:
            raise ValueError("strength must be nonnegative")
        if len(masks) > 64:
            raise ValueError("at most 64 views per view set")
        self.grid = grid
        self.n = grid.size
        self.L = len(masks)
        self.strength = float(strength)
        self.dtype = dtype
        self.device = device or default_device()
        bits = np.zeros(self.n, dtype=np.uint64)
        for v, m in enumerate(masks):
            bits |= np.asarray(m, dtype=np.uint64) << np.uint64(v)
        self.masks_host = [np.asarray(m, dtype=bool) for m in masks]
        self.bits = torch.from_numpy(bits.view(np.int64)).to(self.device)
        self.y = torch.zeros(self.L, self.n, dtype=dtype, device=self.device)
        self._dims = (C.c_int64 * 3)(*grid.dims3)
        self._lib = _abi.load_library()
        self._ctx = _abi.ctx_for(self.device)
        self._code = _abi.dtype_code(dtype)

    # -- primitive device ops ------------------------------------------------
    def _stream(self):
        return _abi.stream_ptr(self.device)

    def _axes(self, x, fn):
        # ping-pong between two fresh buffers; the input is never written
        src = x.contiguous()
        bufs = [torch.empty_like(src), None]
        out = src
        for axis in range(self.grid.ndim):
            if self.grid.dims[axis] == 1:
                continue
            dst = bufs[0] if out is not bufs[0] else (bufs[1] if bufs[1] is not None else torch.empty_like(src))
            if dst is not bufs[0]:
                bufs[1] = dst
            fn(axis, out, dst)
            out = dst
        return out if out is not src else src.clone()

    def _dct(self, x, inverse=False):
        def run(axis, a, b):
            _abi.check(self._lib.bq_dct_axis(self._ctx, self._code, self._dims, axis, int(inverse), a.data_ptr(),
                                             b.data_ptr(), self._stream()), "dct")
        return self._axes(x, run)

    def _smooth(self, x):
        def run(axis, a, b):
            _abi.check(self._lib.bq_smooth_axis(self._ctx, self._code, self._dims, axis, a.data_ptr(), b.data_ptr(),
                                                self._stream()), "smooth")
        return self._axes(x, run)

    def _pw(self, op, x=None, a=None, b=None, s=0.0):
        ref = x if x is not None else a
        out = torch.empty_like(ref)
        _abi.check(self._lib.bq_pointwise(self._ctx, self._code, op, self.n, _abi.ptr(x), _abi.ptr(a), _abi.ptr(b),
                                          float(s), out.data_ptr(), self._stream()), "pointwise")
        return out

    def _vid(self, views):
        """Device view-id list, cached per subset (no host-to-device copy per call,
        so a subset gradient can be captured in a CUDA graph)."""
        key = tuple(views)
        cache = self.__dict__.setdefault("_vid_cache", {})
        if key not in cache:
            cache[key] = torch.tensor(views, dtype=torch.int32, device=self.device)
        return cache[key]

    def _combine(self, F, views, scale, want_r=True, want_cost=False):
        views = list(views)
        vid = self._vid(views)
        ys = _abi.ptr_array([self.y[v] for v in views])
        r = torch.empty_like(F) if want_r else None
        cost = torch.empty(len(views), dtype=torch.float64, device=self.device) if want_cost else None
        _abi.check(self._lib.bq_views_combine(self._ctx, self._code, self.n, F.data_ptr(), ys, self.bits.data_ptr(),
                                              vid.data_ptr(), len(views), float(scale), _abi.ptr(r), _abi.ptr(cost),
                                              self._stream()), "views_combine")
        self._keep = vid
        return r, cost

    def _mask(self, v):
        """View v's 0/1 mask on the device, uploaded once per view (not per call)."""
        cache = self.__dict__.setdefault("_mask_cache", {})
        if v not in cache:
            cache[v] = torch.from_numpy(self.masks_host[v].astype(np.float64)).to(self.device, self.dtype)
        return cache[v]

    # -- the reference's closures (forward_models.py:166-183) -------------
    def fmap(self, x):
        if self.strength == 0.0:
            return x
        return self._pw(0, x=x, a=self._smooth(x), s=self.strength)

    def spectrum(self, x):
        """F = DCT(x + s (Ax)^2): view-independent part of H."""
        return self._dct(self.fmap(x))

    def forward(self, v, x):
        return self._dct(self.fmap(x)) * self._mask(v)

    def jvp(self, v, x, w):
        if self.strength == 0.0:
            inner = w
        else:
            inner = self._pw(1, x=w, a=self._smooth(x), b=self._smooth(w), s=self.strength)
        return self._dct(inner) * self._mask(v)

    def adjoint_tail(self, x, q):
        """q + 2 s A((Ax) . q): the view-independent chain-rule tail of the VJP."""
        if self.strength == 0.0:
            return q
        ax = self._smooth(x)
        return self._pw(3, x=q, b=self._smooth(self._pw(2, a=ax, b=q)), s=self.strength)

    def vjp(self, v, x, z):
        q = self._dct(z * self._mask(v), inverse=True)
        return self.adjoint_tail(x, q)

    # -- batched subset operations ------------------------------------------
    def subset_gradient(self, views, x):
        """(1/|S|) sum_rho J^T (M_rho F - y_rho) with one DCT pair for the subset."""
        F = self.spectrum(x)
        r, _ = self._combine(F, views, 1.0 / len(views))
        return self.adjoint_tail(x, self._dct(r, inverse=True))

    def gauss_newton_subset(self, views, x, v):
        """(1/|S|) sum_rho J_rho^T J_rho v (solvers.py:176-181), one DCT pair per call:
        J_rho v = M_rho DCT(inner(v)) and M_rho^2 = M_rho."""
        if self.strength == 0.0:
            inner = v
        else:
            inner = self._pw(1, x=v, a=self._smooth(x), b=self._smooth(v), s=self.strength)
        G = self._dct(inner)
        zero = torch.zeros_like(G)
        saved = self.y
        self.y = zero.expand(self.L, -1)
        try:
            r, _ = self._combine(G, views, 1.0 / len(views))
        finally:
            self.y = saved
        return self.adjoint_tail(x, self._dct(r, inverse=True))

    def mean_adjoint_measurements(self, views):
        """(1/L) sum_rho J_rho(0)^T y_rho (solvers.py:192-199)."""
        zero = torch.zeros(self.n, dtype=self.dtype, device=self.device)
        r, _ = self._combine(zero, views, -1.0 / len(views))
        return self._dct(r, inverse=True)

    def costs(self, views, x):
        """Device vector of 1/2 ||H_rho(x) - y_rho||^2 for rho in views."""
        F = self.spectrum(x)
        _, c = self._combine(F, views, 1.0, want_r=False, want_cost=True)
        return c


class ViewProblem:
    """One data-fidelity term 1/2 ||H(x) - y||^2 (forward_models.py:25-83).

    Either wraps user callables (as the reference does) or a view of a
    ``DctViewSet`` (device operators)."""

    def __init__(self, forward, jacobian_vec, adjoint_vec, y, view_id=0):
        self._forward = forward
        self._jacobian_vec = jacobian_vec
        self._adjoint_vec = adjoint_vec
        self.y = np.asarray(y, dtype=float)
        self.view_id = int(view_id)
        self.viewset = None

    @classmethod
    def from_viewset(cls, vs: DctViewSet, v: int):
        obj = cls.__new__(cls)
        obj.viewset = vs
        obj.view_id = int(v)
        obj._forward = obj._jacobian_vec = obj._adjoint_vec = None
        return obj

    @property
    def y_device(self):
        return self.viewset.y[self.view_id]

    def __getattr__(self, name):
        if name == "y" and self.__dict__.get("viewset") is not None:
            return self.viewset.y[self.view_id].detach().cpu().numpy()
        raise AttributeError(name)

    def _dev(self, x):
        vs = self.viewset
        return to_dev(x, vs.dtype, vs.device)

    def forward(self, x):
        if self.viewset is None:
            return self._forward(np.asarray(x, dtype=float))
        return out_like(x, self.viewset.forward(self.view_id, self._dev(x)))

    def jacobian_vec(self, x, v):
        if self.viewset is None:
            return self._jacobian_vec(np.asarray(x, dtype=float), np.asarray(v, dtype=float))
        return out_like(v, self.viewset.jvp(self.view_id, self._dev(x), self._dev(v)))

    def adjoint_vec(self, x, z):
        if self.viewset is None:
            return self._adjoint_vec(np.asarray(x, dtype=float), np.asarray(z, dtype=float))
        return out_like(z, self.viewset.vjp(self.view_id, self._dev(x), self._dev(z)))

    def value(self, x):
        if self.viewset is None:
            r = self.forward(x) - self.y
            return 0.5 * float(np.dot(r, r))
        return float(self.viewset.costs([self.view_id], self._dev(x))[0].item())

    def gradient(self, x):
        if self.viewset is None:
            return self.adjoint_vec(x, self.forward(x) - self.y)
        return out_like(x, self.viewset.subset_gradient([self.view_id], self._dev(x)))

    def self_check(self, n, rng, adj_tol=1e-10, grad_tol=1e-4, check=True):
        """Adjoint and finite-difference tests (forward_models.py:66-83); the
        RNG is consumed exactly like the reference even when check=False."""
        x = rng.standard_normal(n)
        v = rng.standard_normal(n)
        m = n if self.viewset is not None else self.y.shape[0]
        z = rng.standard_normal(m)
        d = None
        if not check:
            rng.standard_normal(n)
            return
        lhs = float(np.dot(self.jacobian_vec(x, v), z))
        rhs = float(np.dot(v, self.adjoint_vec(x, z)))
        scale = max(1.0, abs(lhs), abs(rhs))
        if abs(lhs - rhs) > adj_tol * scale:
            raise RuntimeError(f"view {self.view_id}: adjoint test failed ({lhs} vs {rhs})")
        g = self.gradient(x)
        h = 1e-6
        d = rng.standard_normal(n)
        d /= np.linalg.norm(d)
        fd = (self.value(x + h * d) - self.value(x - h * d)) / (2 * h)
        an = float(np.dot(g, d))
        if abs(fd - an) > grad_tol * max(1.0, abs(fd), abs(an)):
            raise RuntimeError(f"view {self.view_id}: gradient test failed ({an} vs {fd})")


def _make_views(grid, n_views, mask_fraction, seed, strength, x_gt, noise_snr_db, dtype=torch.float64,
                self_check=True, device=None):
    if strength < 0:
        raise ValueError("strength must be nonnegative")
    rng = np.random.default_rng(seed)
    if x_gt is None:
        x_gt = make_phantom(grid, seed=seed).values
    x_gt = np.asarray(x_gt, dtype=float)
    masks, _ = spectrum_masks(grid, n_views, mask_fraction)
    vs = DctViewSet(grid, masks, strength=strength, dtype=dtype, device=device)
    F = vs.spectrum(to_dev(x_gt, dtype, vs.device))
    views = []
    for v in range(n_views):
        y = F * vs._mask(v)
        if noise_snr_db is not None:
            noise = rng.standard_normal(grid.size) * masks[v].astype(float)
            power = np.linalg.norm(noise)
            if power > 0:
                ynorm = float(torch.linalg.vector_norm(y.double()).item())
                noise *= ynorm / power * 10.0 ** (-noise_snr_db / 20.0)
            y = y + to_dev(noise, dtype, vs.device)
        vs.y[v] = y
        view = ViewProblem.from_viewset(vs, v)
        view.self_check(grid.size, rng, check=self_check)
        views.append(view)
    return views


def make_linear_views(grid, n_views, mask_fraction=0.5, seed=0, x_gt=None, noise_snr_db=None, **kw):
    return _make_views(grid, n_views, mask_fraction, seed, 0.0, x_gt, noise_snr_db, **kw)


def make_nonlinear_views(grid, n_views, strength=0.1, mask_fraction=0.5, seed=0, x_gt=None, noise_snr_db=None,
                         **kw):
    return _make_views(grid, n_views, mask_fraction, seed, strength, x_gt, noise_snr_db, **kw)


# ---------------------------------------------------------------------------
# subset / full costs (forward_models.py:286-309)
# ---------------------------------------------------------------------------
def _shared_viewset(views, indices):
    vs = getattr(views[indices[0]], "viewset", None) if len(indices) else None
    if vs is None or any(getattr(views[i], "viewset", None) is not vs for i in indices):
        return None
    return vs


def subset_gradient_async(views, indices, x):
    """Device subset gradient (torch in, torch out) for views of one DctViewSet."""
    idx = [int(i) for i in indices]
    vs = _shared_viewset(views, idx)
    if vs is None:
        raise ValueError("device subset gradient needs views of one DctViewSet")
    return vs.subset_gradient([views[i].view_id for i in idx], x)


def subset_gradient(views, indices, x):
    idx = [int(i) for i in indices]
    vs = _shared_viewset(views, idx)
    if vs is not None:
        return out_like(x, vs.subset_gradient([views[i].view_id for i in idx], to_dev(x, vs.dtype, vs.device)))
    g = np.zeros_like(np.asarray(x, dtype=float))
    for i in idx:
        g += views[i].gradient(x)
    return g / len(idx)


def subset_value(views, indices, x):
    idx = [int(i) for i in indices]
    vs = _shared_viewset(views, idx)
    if vs is not None:
        c = vs.costs([views[i].view_id for i in idx], to_dev(x, vs.dtype, vs.device))
        return float(c.sum().item()) / len(idx)
    return sum(views[i].value(x) for i in idx) / len(idx)


def data_fidelity(views, x):
    return subset_value(views, list(range(len(views))), x)


def full_cost(views, x, tv_weight, grid, mode=TvMode.ISOTROPIC):
    cost = data_fidelity(views, x)
    if tv_weight:
        cost += tv_weight * tv_value(grid, x, mode)
    return cost


__all__ = [
    "ViewProblem",
    "DctViewSet",
    "Phantom",
    "spectrum_masks",
    "make_linear_views",
    "make_nonlinear_views",
    "make_phantom",
    "snr_db",
    "data_fidelity",
    "full_cost",
    "subset_value",
    "subset_gradient",
    "subset_gradient_async",
]

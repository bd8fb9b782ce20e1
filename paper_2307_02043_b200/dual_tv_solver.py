"""Weighted constrained TV prox on the device — drop-in for ``tvqn.dual_tv_solver``.

Reference: ``/root/reference/pkg/src/tvqn/dual_tv_solver.py``
  * ``DualTvProblem`` (:25-79): same fields, defaults and validation; omega
    defaults to 1/tau (scalar metric) or to the bound of
    ``DiagPlusLowRank.default_omega`` (per-voxel diagonal, D-6).
  * ``DualSolveReport`` (:82-92): same fields.
  * ``dual_step_size`` (:155-158): 1 / (4 ndim omega reg).
  * ``solve(prob, eps=1e-5, max_iter=100, accelerated=True)`` (:161-250):
    ONE ``bq_wtv_prox`` launch (persistent cooperative kernel running the FGP
    loop, the Woodbury shift, the semi-smooth Newton, the projection and the
    momentum, with every stop/accept decision on the device).

numpy inputs give numpy outputs (float64 compute); torch CUDA inputs give
torch outputs in their dtype (float32 or float64); the arithmetic runs in the
metric's dtype (where U and d live), v is cast to it.  ``solve_async`` is the
GPU-resident variant that leaves the report on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from ._tensors import is_torch, out_like, to_dev
from .tv_ops import Grid, TvMode, dual_adjoint, dual_divergence, tv_value
from .wpm import BoxSet, DiagPlusLowRank, apply_metric, apply_metric_inverse, wpm_box


@dataclass
class DualTvProblem:
    grid: Grid
    v: object
    w: DiagPlusLowRank
    reg: float
    mode: TvMode = TvMode.ISOTROPIC
    box: BoxSet = field(default_factory=BoxSet)
    omega: float = None
    warm_start: object = None
    beta_warm: object = None
    newton_eps: float = 1e-6
    newton_max_iter: int = 50

    def __post_init__(self):
        if self.reg < 0:
            raise ValueError("reg must be nonnegative")
        if self.omega is None:
            self.omega = self.w.default_omega()
        if not self.omega > 0:
            raise ValueError("omega must be positive")
        if self.beta_warm is not None and not is_torch(self.beta_warm):
            self.beta_warm = np.asarray(self.beta_warm, dtype=float)
        self.mode = TvMode.parse(self.mode)


@dataclass
class DualSolveReport:
    x: object
    p_star: object
    iterations: int
    rel_change: float
    converged: bool
    newton_iterations: int = 0
    beta_star: object = None


def metric_min_eig_inverse(w: DiagPlusLowRank, iters=50, seed=0):
    """1/lambda_min(W) by inverse power iteration through the device Woodbury
    inverse (dual_tv_solver.py:95-116)."""
    n = w.dim
    if n == 0 or w.rank == 0:
        return 1.0 / w.tau if w.d is None else w.default_omega()
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    vt = to_dev(v, w.dtype, w.device)
    mu = 1.0 / w.tau if w.d is None else w.default_omega()
    for _ in range(iters):
        z = apply_metric_inverse(w, vt)
        mu = float(torch.dot(vt.double(), z.double()).item())
        nz = float(torch.linalg.vector_norm(z.double()).item())
        if nz == 0.0:
            break
        vt = z / nz
    return mu


def _w_of_p_dev(prob: DualTvProblem, p) -> torch.Tensor:
    v = to_dev(prob.v, prob.w.dtype, prob.w.device)
    if prob.reg == 0.0:
        return v
    pt = to_dev(p, prob.w.dtype, prob.w.device)
    return v - prob.reg * apply_metric_inverse(prob.w, dual_divergence(prob.grid, pt))


def w_of_p(prob: DualTvProblem, p):
    """Centre shift w(P) = v - reg W^-1 d(P) (dual_tv_solver.py:119-123), on the device."""
    if prob.reg == 0.0 and not is_torch(prob.v):
        return np.asarray(prob.v, dtype=float)
    return out_like(prob.v, _w_of_p_dev(prob, p))


def _prox_of(prob: DualTvProblem, p, beta0=None):
    """(q, info) with q a device tensor."""
    return wpm_box(_w_of_p_dev(prob, p), prob.w, prob.box, beta0=beta0, eps=prob.newton_eps,
                   max_iter=prob.newton_max_iter, full_output=True)


def dual_gradient(prob: DualTvProblem, p):
    """-2 reg [D^1 q; ...; D^d q], q = wpm_box(w(P)) (dual_tv_solver.py:138-144)."""
    if prob.reg == 0.0:
        z = torch.zeros(prob.grid.ndim, prob.grid.size, dtype=prob.w.dtype, device=prob.w.device)
        return out_like(prob.v, z)
    q, _ = _prox_of(prob, to_dev(p, prob.w.dtype, prob.w.device))
    return out_like(prob.v, -2.0 * prob.reg * dual_adjoint(prob.grid, q))


def dual_objective(prob: DualTvProblem, p):
    """||w(P)||_W^2 - ||w(P) - prox(w(P))||_W^2 (dual_tv_solver.py:147-152)."""
    wp = _w_of_p_dev(prob, p)
    q, _ = _prox_of(prob, to_dev(p, prob.w.dtype, prob.w.device))
    diff = wp - q
    a = torch.dot(wp.double(), apply_metric(prob.w, wp).double())
    b = torch.dot(diff.double(), apply_metric(prob.w, diff).double())
    return float((a - b).item())


def primal_objective(prob: DualTvProblem, x):
    """1/2 ||x - v||_W^2 + reg TV(x) (dual_tv_solver.py:253-260)."""
    xt = to_dev(x, prob.w.dtype, prob.w.device)
    diff = xt - to_dev(prob.v, prob.w.dtype, prob.w.device)
    quad = 0.5 * float(torch.dot(diff.double(), apply_metric(prob.w, diff).double()).item())
    return quad + prob.reg * tv_value(prob.grid, xt, prob.mode)


def dual_step_size(prob: DualTvProblem) -> float:
    return 1.0 / (4.0 * prob.grid.ndim * prob.omega * prob.reg)


class ProxWorkspace:
    """Reusable device buffers for repeated solves on one grid (no allocation per call)."""

    def __init__(self, grid: Grid, dtype, device):
        n, d = grid.size, grid.ndim
        self.grid, self.dtype, self.device = grid, dtype, device
        self.p = torch.zeros(d, n, dtype=dtype, device=device)
        self.pb = torch.empty(d, n, dtype=dtype, device=device)
        self.p2 = torch.empty(d, n, dtype=dtype, device=device)  # third slot of the P ring (fused kernel)
        self.a = torch.empty(n, dtype=dtype, device=device)
        self.a2 = torch.empty(n, dtype=dtype, device=device)
        self.x = torch.empty(n, dtype=dtype, device=device)
        self.beta = torch.zeros(_abi.BQ_MAX_RANK, dtype=torch.float64, device=device)
        self.report = torch.zeros(_abi.REPORT_BYTES, dtype=torch.uint8, device=device)


def _launch(prob: DualTvProblem, v: torch.Tensor, ws: ProxWorkspace, eps, max_iter, accelerated):
    g, w = prob.grid, prob.w
    if v.numel() != g.size:
        raise ValueError(f"expected {g.size} entries, got {v.numel()}")
    if w.rank and w.dim != g.size:
        raise ValueError(f"dimension mismatch: metric is {w.dim}, grid is {g.size}")
    if (w.rank or w.d is not None) and w.dtype != ws.dtype:
        # the kernel reads U and d in the descriptor's dtype
        raise ValueError(f"metric dtype {w.dtype} differs from the workspace dtype {ws.dtype}")
    lo, hi, lo_a, hi_a = prob.box.device_args(ws.dtype, ws.device)
    desc = _abi.WtvDesc()
    desc.ndim = g.ndim
    desc.dtype = _abi.dtype_code(ws.dtype)
    desc.dims[:] = g.dims3
    desc.mode = prob.mode.code
    desc.rank = w.rank
    desc.sign = w.sign
    desc.accelerated = int(bool(accelerated))
    desc.tau = w.tau if w.d is None else 0.0
    desc.reg = float(prob.reg)
    desc.step = dual_step_size(prob) if prob.reg > 0 else 0.0
    desc.eps = float(eps)
    desc.max_iter = int(max_iter)
    desc.newton_max_iter = int(prob.newton_max_iter)
    desc.newton_eps = float(prob.newton_eps)
    desc.lo, desc.hi = lo, hi
    desc.lo_arr, desc.hi_arr = _abi.ptr(lo_a), _abi.ptr(hi_a)
    desc.d = _abi.ptr(w.d)
    desc.U = w.Ut.data_ptr() if w.rank else None
    desc.v = v.data_ptr()
    desc.p, desc.pb, desc.a, desc.x = ws.p.data_ptr(), ws.pb.data_ptr(), ws.a.data_ptr(), ws.x.data_ptr()
    desc.beta = ws.beta.data_ptr()
    desc.report = ws.report.data_ptr()
    desc.p2 = ws.p2.data_ptr()
    desc.a2 = ws.a2.data_ptr()
    lib = _abi.load_library()
    _abi.check(lib.bq_wtv_prox(_abi.ctx_for(ws.device), desc, _abi.stream_ptr(ws.device)), "solve")
    # keep optional temporaries alive until the stream has consumed them
    ws._keep = (lo_a, hi_a, v)


def _check_args(prob, eps, max_iter):
    if eps <= 0:
        raise ValueError("eps must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")


def solve_async(prob: DualTvProblem, ws: ProxWorkspace, eps=1e-5, max_iter=100, accelerated=True,
                load_warm=True):
    """GPU-resident solve: reads v/warm start from ``prob`` (torch), writes ws.x,
    ws.p (P*), ws.beta (beta*) and the device report.  No host sync."""
    _check_args(prob, eps, max_iter)
    v = to_dev(prob.v, ws.dtype, ws.device)
    d, n = prob.grid.ndim, prob.grid.size
    if load_warm:
        if prob.warm_start is not None:
            p0 = to_dev(prob.warm_start, ws.dtype, ws.device)
            if p0.numel() != d * n or (not is_torch(prob.warm_start) and np.shape(prob.warm_start) != (d, n)):
                raise ValueError(f"warm start must have shape {(d, n)}")
            ws.p.copy_(p0.reshape(d, n))
        else:
            ws.p.zero_()
        ws.beta.zero_()
        bw = prob.beta_warm
        if bw is not None and np.shape(bw)[0] == prob.w.rank and prob.w.rank:
            ws.beta[: prob.w.rank] = to_dev(bw, torch.float64, ws.device)
    _launch(prob, v, ws, eps, max_iter, accelerated)
    return ws


def read_report(ws: ProxWorkspace) -> _abi.WtvReport:
    rep = _abi.WtvReport.from_buffer_copy(ws.report.cpu().numpy().tobytes())
    if rep.status:
        _abi.check(rep.status, "solve")
    return rep


def solve(prob: DualTvProblem, eps=1e-5, max_iter=100, accelerated=True) -> DualSolveReport:
    """Drop-in for ``tvqn.dual_tv_solver.solve`` (dual_tv_solver.py:161-250)."""
    _check_args(prob, eps, max_iter)
    # compute in the metric's dtype (U and d live there); v is cast to it and
    # torch outputs come back in v's own dtype
    dtype = prob.w.dtype
    ws = ProxWorkspace(prob.grid, dtype, prob.w.device)
    solve_async(prob, ws, eps, max_iter, accelerated)
    rep = read_report(ws)
    r = prob.w.rank
    like = prob.v
    beta = ws.beta[:r]
    if prob.reg == 0.0:
        p_star = prob.warm_start if prob.warm_start is not None else out_like(like, torch.zeros_like(ws.p))
        if not is_torch(like) and prob.warm_start is not None:
            p_star = np.asarray(prob.warm_start)
    else:
        p_star = out_like(like, ws.p)
    if is_torch(like) and like.dtype in (torch.float32, torch.float64) and like.dtype != dtype:
        ws.x, ws.p = ws.x.to(like.dtype), ws.p.to(like.dtype)
        if prob.reg != 0.0:
            p_star = ws.p
    return DualSolveReport(
        x=out_like(like, ws.x),
        p_star=p_star,
        iterations=int(rep.iterations),
        rel_change=float(rep.rel_change),
        converged=bool(rep.converged),
        newton_iterations=int(rep.newton_iterations),
        beta_star=out_like(like, beta) if r else (np.zeros(0) if not is_torch(like) else beta),
    )


__all__ = ["DualTvProblem", "DualSolveReport", "metric_min_eig_inverse", "w_of_p", "dual_gradient",
           "dual_objective", "dual_step_size", "solve", "primal_objective", "solve_async", "ProxWorkspace",
           "read_report"]

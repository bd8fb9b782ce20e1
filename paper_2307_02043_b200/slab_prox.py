"""z-slab-sharded weighted-TV prox (north star (4); config 5).

The FGP dual iteration of ``tvqn.dual_tv_solver.solve``
(``/root/reference/pkg/src/tvqn/dual_tv_solver.py:161-250``) with its
structured projection (``wpm.py:145-253``) over a 3-D volume split along
dims[2] into contiguous slabs of planes, one slab per GPU.  Per FGP
iteration and rank (``csrc/slab_prox.cu`` passes, host control here):

  1. ``bq_slab_div``    t = D^-1 div(Pbar) over the slab; needs Pbar_z of the
                        plane just below the slab (1-plane halo from rank-1)
                        -> all-reduce s = U^T t (r doubles); c = cap^-1 s
  2. ``bq_slab_newton`` Newton residual / Jacobian at beta -> all-reduce of
                        r + r(r+1)/2 doubles per Newton step; the controller
                        (accept, best residual, Levenberg) runs identically
                        on every rank on the all-reduced scalars
  3. ``bq_slab_q``      q = clamp(z(beta*)); q of the plane just above the slab
                        comes from rank+1 (1-plane halo)
  4. ``bq_slab_dual``   P_next, Pbar_next and the two norms -> all-reduce of 2
                        doubles; the rel-change stop and the FISTA t-sequence
                        are decided on the all-reduced values

Communication budget per FGP iteration at K1 x K2 planes of s-byte words:
two halo planes (Pbar_z up, q down; 2 K1 K2 s bytes each way), and
2 + (newton steps + 1) all-reduces of <= 46 doubles.  At 256^3 fp32 the
halos are 256 KB per neighbour per iteration.

Sharding is by slabs of one process: ``SlabGroup`` holds the slabs this
process owns (one per rank under torchrun; several in one process for the
single-GPU loopback test) and reduces their partials locally before the
cross-process all-reduce, so the same control code runs in every layout.
The per-slab compute is a backend object: ``DeviceSlabs`` (libbq, the
product path) -- the CPU tests plug a numpy backend into the same control
code to check it with gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _abi
from ._tensors import to_dev
from .tv_ops import TvMode

_LEVENBERG = 1e-8  # wpm.py:21


def slab_bounds(k3: int, world: int):
    """Contiguous plane ranges [z0, z1) per rank (sizes differ by <= 1)."""
    base, extra = divmod(k3, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((z, z + n))
        z += n
    return out


@dataclass
class SlabReport:
    x: torch.Tensor            # this process's slabs of x, concatenated along z
    p_star: torch.Tensor       # (3, local N)
    iterations: int
    rel_change: float
    converged: bool
    newton_iterations: int
    beta_star: np.ndarray


class Comm:
    """Cross-process steps: all-reduce(sum) of small vectors, plane exchange with
    the neighbouring ranks.  world == 1 (or no process group): no-ops."""

    def __init__(self, group=None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1

    def _host_staged(self, t):
        # gloo (the CPU tests, and bench.py's one-GPU functional mode) moves host tensors
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            if self._host_staged(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _peer(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def shift(self, send: torch.Tensor, recv: torch.Tensor, up: bool):
        """Send `send` to rank+1 (up) or rank-1 (down) and receive the matching plane
        from the opposite neighbour into `recv` (edge ranks skip the missing side)."""
        if self.world == 1:
            return
        ops = []
        dst = self.rank + 1 if up else self.rank - 1
        src = self.rank - 1 if up else self.rank + 1
        staged = self._host_staged(recv)
        snd = send.cpu() if staged else send.contiguous()
        rcv = torch.empty(recv.shape, dtype=recv.dtype) if staged else recv
        if 0 <= dst < self.world:
            ops.append(dist.P2POp(dist.isend, snd, self._peer(dst), self.group))
        if 0 <= src < self.world:
            ops.append(dist.P2POp(dist.irecv, rcv, self._peer(src), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if staged and 0 <= src < self.world:
            recv.copy_(rcv)


class SlabGroup:
    """The slabs one process owns, with their global placement.

    `slabs` are consecutive in z; slab i of this process covers planes
    bounds[i].  A backend implements the four passes on one slab."""

    def __init__(self, backend, comm: Comm, dims, bounds, k3):
        self.be, self.comm = backend, comm
        self.dims, self.bounds, self.k3 = tuple(dims), list(bounds), int(k3)
        self.plane = dims[0] * dims[1]

    # ---- cross-slab plumbing -------------------------------------------------
    def reduce(self, parts):
        """Sum of per-slab partial vectors (local slab order), then across ranks."""
        tot = parts[0].clone()
        for p in parts[1:]:
            tot += p
        return self.comm.allreduce(tot)

    def halo_up(self, planes):
        """planes[i] = the top plane slab i sends upward; returns, per slab, the plane
        received from below (None for the global first slab)."""
        n = len(planes)
        out = [None] * n
        for i in range(1, n):
            out[i] = planes[i - 1]
        if self.comm.world > 1:
            recv = torch.empty_like(planes[0])
            self.comm.shift(planes[-1], recv, up=True)
            if self.bounds[0][0] > 0:
                out[0] = recv
        return out

    def halo_down(self, planes):
        """planes[i] = the bottom plane slab i sends downward; returns, per slab, the
        plane received from above (None for the global last slab)."""
        n = len(planes)
        out = [None] * n
        for i in range(n - 1):
            out[i] = planes[i + 1]
        if self.comm.world > 1:
            recv = torch.empty_like(planes[0])
            self.comm.shift(planes[0], recv, up=False)
            if self.bounds[-1][1] < self.k3:
                out[-1] = recv
        return out


# control-block layout (bq_slab_ctl, include/bq.h)
C_DONE, C_IT, C_BEST, C_TOTAL, C_REL, C_FGP, C_LAST, C_BETA = 0, 1, 2, 3, 4, 5, 6, 8
OP_INIT, OP_COEF, OP_NEWTON, OP_NORMS, OP_UNDO = 0, 1, 2, 3, 4


def slab_solve(sg: SlabGroup, *, rank, sign, tau, scalar, gram, reg, step, eps=1e-5, max_iter=100,
               accelerated=True, newton_eps=1e-6, newton_max_iter=50, beta0=None, p0=None, spec=2):
    """FGP loop of dual_tv_solver.py:161-250 over the slabs of `sg` (every rank
    calls it with its own slabs).

    The scalar control (Woodbury coefficient, the semi-smooth Newton of
    wpm.py:170-231, the rel-change stop) runs in the backend's control block
    on the all-reduced sums, so the passes, the all-reduces and the control
    steps are all stream-ordered.  The host reads the control block once per
    FGP iteration, after `spec` speculative Newton evaluations (more only when
    the Newton needs them); the next iteration's divergence and Newton are
    queued before the host learns whether the current one met the stop test,
    and are undone (beta, Newton count) when it did."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    be = sg.be
    ns = len(sg.bounds)
    beta = np.zeros(rank) if (beta0 is None or np.shape(beta0)[0] != rank) else np.asarray(beta0, float).copy()
    init = np.zeros(72)
    if rank:
        cap = np.eye(rank) + sign * (gram / tau if scalar else gram)
        init[: rank * rank] = np.linalg.cholesky(cap).reshape(-1)
        init[64:64 + rank] = beta
    be.ctl(OP_INIT, init, newton_eps, newton_max_iter, eps)

    def div_coef(field):
        """t = D^-1 div(field) per slab, then c = cap^-1 U^T t and a Newton reset."""
        if reg == 0.0:
            t = [be.zeros(s) for s in range(ns)]
            be.ctl(OP_COEF, np.zeros(max(rank, 1)), newton_eps, newton_max_iter, eps)
            return t
        halos = sg.halo_up([be.top_plane_z(field[s]) for s in range(ns)])
        out = [be.div(s, field[s], halos[s]) for s in range(ns)]
        sv = sg.reduce([o[1] for o in out]) if rank else np.zeros(1)
        be.ctl(OP_COEF, sv, newton_eps, newton_max_iter, eps)
        return [o[0] for o in out]

    def newton_evals(t, count):
        for _ in range(count if rank else 0):
            part = sg.reduce([be.newton(s, t[s]) for s in range(ns)])
            be.ctl(OP_NEWTON, part, newton_eps, newton_max_iter, eps)

    def finish(t, c):
        while c[C_DONE] == 0.0:
            newton_evals(t, 1)
            c = be.read_ctl()
        return c

    p = [be.dual_field(s, None if p0 is None else p0[s]) for s in range(ns)]
    if reg == 0.0:
        t = div_coef(p)
        newton_evals(t, spec)
        c = finish(t, be.read_ctl())
        q = [be.q(s, t[s]) for s in range(ns)]
        return SlabReport(x=be.concat(q), p_star=be.concat_dual(p), iterations=1, rel_change=0.0, converged=True,
                          newton_iterations=int(c[C_TOTAL]), beta_star=np.array(c[C_BETA:C_BETA + rank]))
    pbar = [x.clone() for x in p]
    tk = 1.0
    converged = False
    iterations = 0
    t = div_coef(pbar)
    newton_evals(t, spec)
    for it in range(1, max_iter + 1):
        c = be.read_ctl()  # the one host read of the iteration
        if it > 1 and c[C_FGP] != 0.0:  # iteration it-1 met the stop test: drop the speculative one
            be.ctl(OP_UNDO, None, newton_eps, newton_max_iter, eps)
            converged = True
            break
        iterations = it
        finish(t, c)
        q = [be.q(s, t[s]) for s in range(ns)]
        qh = sg.halo_down([be.bottom_plane(q[s]) for s in range(ns)])
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * tk * tk))
        mom = (tk - 1.0) / t_next if accelerated else 0.0
        outs = [be.dual(s, pbar[s], p[s], q[s], qh[s], step, mom) for s in range(ns)]
        be.ctl(OP_NORMS, sg.reduce([o[2] for o in outs]), newton_eps, newton_max_iter, eps)
        p = [o[0] for o in outs]
        pbar = [o[1] for o in outs]
        if accelerated:
            tk = t_next
        if it < max_iter:
            t = div_coef(pbar)
            newton_evals(t, spec)
    c = be.read_ctl()
    if not converged and c[C_FGP] != 0.0:  # the last iteration met the stop test
        converged = True
    rel = float(c[C_REL])
    # final prox at P (dual_tv_solver.py:240-241)
    t = div_coef(p)
    newton_evals(t, spec)
    c = finish(t, be.read_ctl())
    q = [be.q(s, t[s]) for s in range(ns)]
    return SlabReport(x=be.concat(q), p_star=be.concat_dual(p), iterations=iterations, rel_change=rel,
                      converged=converged, newton_iterations=int(c[C_TOTAL]),
                      beta_star=np.array(c[C_BETA:C_BETA + rank]))


class DeviceSlabs:
    """libbq passes (csrc/slab_prox.cu) on this process's slabs.

    v_parts / d_parts / U_parts: per slab, the local v (N_s), the optional
    per-voxel diagonal (N_s) and U as (rank, N_s) -- device tensors of one
    dtype; planes are contiguous, so a slab is a contiguous range of the
    global flat vector."""

    def __init__(self, dims, bounds, k3, dtype, device, v_parts, U_parts, d_parts=None, *, rank, sign, tau, reg,
                 lo, hi, mode=TvMode.ISOTROPIC):
        self.K1, self.K2 = int(dims[0]), int(dims[1])
        self.plane = self.K1 * self.K2
        self.dtype, self.device = dtype, device
        self.lib = _abi.load_library()
        self.ctx = _abi.ctx_for(device)
        self.v = [to_dev(v, dtype, device) for v in v_parts]
        self.U = [to_dev(u, dtype, device).reshape(rank, -1).contiguous() if rank else None for u in U_parts]
        self.d = [to_dev(d, dtype, device) if d is not None else None for d in (d_parts or [None] * len(bounds))]
        self.descs = []
        for s, (z0, z1) in enumerate(bounds):
            D = _abi.SlabDesc()
            D.dtype = _abi.dtype_code(dtype)
            D.mode = TvMode.parse(mode).code
            D.rank, D.sign = rank, sign
            D.K1, D.K2, D.L = self.K1, self.K2, z1 - z0
            D.first, D.last = int(z0 == 0), int(z1 == k3)
            D.tau = float(tau) if self.d[s] is None else 0.0
            D.reg, D.lo, D.hi = float(reg), float(lo), float(hi)
            D.d = _abi.ptr(self.d[s])
            D.U = _abi.ptr(self.U[s])
            D.v = self.v[s].data_ptr()
            self.descs.append(D)
        self.rank = rank
        self._dots = torch.empty(len(bounds), 64, dtype=torch.float64, device=device)
        self.ctl_buf = torch.zeros(128, dtype=torch.float64, device=device)
        self._in = torch.zeros(72, dtype=torch.float64, device=device)
        self._zeros = torch.zeros(72, dtype=torch.float64, device=device)
        self._host = torch.zeros(128, dtype=torch.float64).pin_memory()
        for D in self.descs:
            D.ctl = self.ctl_buf.data_ptr()

    def _st(self):
        return _abi.stream_ptr(self.device)

    def _n(self, s):
        return self.v[s].numel()

    def zeros(self, s):
        return torch.zeros(self._n(s), dtype=self.dtype, device=self.device)

    def dual_field(self, s, init):
        if init is None:
            return torch.zeros(3, self._n(s), dtype=self.dtype, device=self.device)
        return to_dev(init, self.dtype, self.device).reshape(3, self._n(s)).clone()

    def top_plane_z(self, field):
        return field[2, -self.plane:].contiguous()

    def bottom_plane(self, q):
        return q[: self.plane].contiguous()

    def div(self, s, field, halo):
        t = torch.empty(self._n(s), dtype=self.dtype, device=self.device)
        sv = self._dots[s, :8]
        _abi.check(self.lib.bq_slab_div(self.ctx, self.descs[s], field.data_ptr(), _abi.ptr(halo), t.data_ptr(),
                                        sv.data_ptr() if self.rank else None, self._st()), "slab div")
        return t, sv[: self.rank].clone()

    def newton(self, s, t):
        nv = self.rank + self.rank * (self.rank + 1) // 2
        out = self._dots[s, 8:8 + nv]
        _abi.check(self.lib.bq_slab_newton(self.ctx, self.descs[s], t.data_ptr(), None, None, out.data_ptr(),
                                           self._st()), "slab newton")
        return out.clone()

    def q(self, s, t):
        q = torch.empty(self._n(s), dtype=self.dtype, device=self.device)
        _abi.check(self.lib.bq_slab_q(self.ctx, self.descs[s], t.data_ptr(), None, None, q.data_ptr(), self._st()),
                   "slab q")
        return q

    def ctl(self, op, inp, newton_eps, newton_max_iter, eps):
        """One control step on the (all-reduced) input, stream-ordered (bq_slab_ctl)."""
        ptr = None
        if inp is not None:
            if isinstance(inp, torch.Tensor):
                ptr = inp.data_ptr()
                self._keep = inp
            else:  # host array: INIT (once per solve) or the all-zero rank-0 / reg-0 input
                a = np.asarray(inp, dtype=float)
                if np.any(a):
                    self._in[: len(a)].copy_(torch.as_tensor(a))
                    ptr = self._in.data_ptr()
                else:
                    ptr = self._zeros.data_ptr()
        _abi.check(self.lib.bq_slab_ctl(self.ctx, self.descs[0], int(op), ptr, float(newton_eps),
                                        int(newton_max_iter), float(eps), self._st()), "slab ctl")

    def read_ctl(self):
        self._host.copy_(self.ctl_buf, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self._host.numpy()

    def dual(self, s, pbar, p, q, halo, step, mom):
        pn = torch.empty_like(p)
        pbn = torch.empty_like(p)
        nrm = self._dots[s, 60:62]
        _abi.check(self.lib.bq_slab_dual(self.ctx, self.descs[s], pbar.data_ptr(), p.data_ptr(), q.data_ptr(),
                                         _abi.ptr(halo), float(step), float(mom), pn.data_ptr(), pbn.data_ptr(),
                                         nrm.data_ptr(), self._st()), "slab dual")
        return pn, pbn, nrm.clone()

    def concat(self, parts):
        return torch.cat(parts)

    def concat_dual(self, parts):
        return torch.cat(parts, dim=1)


def solve_sharded(grid, v, w, reg, box, *, group=None, slabs_per_rank=1, mode=TvMode.ISOTROPIC, omega=None,
                  eps=1e-5, max_iter=100, accelerated=True, newton_eps=1e-6, newton_max_iter=50, beta0=None,
                  dtype=None, device=None):
    sp = ShardedProx(grid, v, w, reg, box, group=group, slabs_per_rank=slabs_per_rank, mode=mode, omega=omega,
                     dtype=dtype, device=device)
    return sp.run(eps=eps, max_iter=max_iter, accelerated=accelerated, newton_eps=newton_eps,
                  newton_max_iter=newton_max_iter, beta0=beta0), sp.bounds


class ShardedProx:
    """Sharded counterpart of ``dual_tv_solver.solve`` for a 3-D grid.

    Every rank of `group` passes the same GLOBAL problem description (grid, and
    v / w / box as full arrays it can slice, or device tensors) and gets back
    its own slabs of x and P*.  `slabs_per_rank` > 1 splits each rank's share
    further (the single-GPU loopback layout).  Box bounds must be scalars.
    Returns (SlabReport, [(z0, z1) per local slab]).  ``ShardedProx`` is the
    reusable form (slabs and device buffers set up once, ``run`` per solve)."""

    def __init__(self, grid, v, w, reg, box, *, group=None, slabs_per_rank=1, mode=TvMode.ISOTROPIC, omega=None,
                 dtype=None, device=None):
        self._setup(grid, v, w, reg, box, group, slabs_per_rank, mode, omega, dtype, device)

    def _setup(self, grid, v, w, reg, box, group, slabs_per_rank, mode, omega, dtype, device):
        if grid.ndim != 3:
            raise ValueError("the z-slab prox shards 3-D grids")
        if isinstance(box.lower, np.ndarray) or isinstance(box.upper, np.ndarray):
            raise ValueError("the z-slab prox takes scalar box bounds")
        comm = Comm(group)
        k1, k2, k3 = grid.dims
        allb = slab_bounds(k3, comm.world * slabs_per_rank)
        mine = allb[comm.rank * slabs_per_rank:(comm.rank + 1) * slabs_per_rank]
        if any(z1 <= z0 for z0, z1 in mine):
            raise ValueError(f"{k3} planes cannot give every slab at least one plane")
        dtype = dtype or w.dtype
        device = device or w.device
        plane = k1 * k2
        vt = to_dev(v, dtype, device)
        v_parts = [vt[z0 * plane:z1 * plane] for z0, z1 in mine]
        U_parts = [w.Ut[:, z0 * plane:z1 * plane] if w.rank else None for z0, z1 in mine]
        d_parts = [w.d[z0 * plane:z1 * plane] for z0, z1 in mine] if w.d is not None else None
        gram = None
        if w.rank:
            gram = w.gram.reshape(w.rank, w.rank).cpu().numpy()  # U^T D^-1 U (global, from the metric)
        be = DeviceSlabs(grid.dims, mine, k3, dtype, device, v_parts, U_parts, d_parts, rank=w.rank, sign=w.sign,
                         tau=w.tau if w.d is None else 1.0, reg=reg, lo=box.lower, hi=box.upper, mode=mode)
        if omega is None:
            omega = w.default_omega()
        self.step = 1.0 / (4.0 * 3 * omega * reg) if reg > 0 else 0.0
        self.sg = SlabGroup(be, comm, grid.dims, mine, k3)
        self.bounds = mine
        self.kw = dict(rank=w.rank, sign=w.sign, tau=w.tau if w.d is None else 1.0, scalar=w.d is None, gram=gram,
                       reg=reg)

    def run(self, eps=1e-5, max_iter=100, accelerated=True, newton_eps=1e-6, newton_max_iter=50, beta0=None):
        return slab_solve(self.sg, step=self.step, eps=eps, max_iter=max_iter, accelerated=accelerated,
                          newton_eps=newton_eps, newton_max_iter=newton_max_iter, beta0=beta0, **self.kw)


__all__ = ["slab_bounds", "Comm", "SlabGroup", "slab_solve", "DeviceSlabs", "solve_sharded", "ShardedProx",
           "SlabReport"]

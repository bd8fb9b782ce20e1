"""GPU-resident BQNPM outer loop with CUDA-graph replay.

The reference loop (``/root/reference/pkg/src/tvqn/solvers.py:253-317``)
takes three host decisions per iteration k > K_s: whether the SR1 step is
usable (``np.any(s)``), whether the SR1 term is accepted (which sets the rank
of the aggregated metric), and -- through ``DiagPlusLowRank`` /
``DualTvProblem`` -- the metric's tau and the dual step.  Here all three stay
on the device:

* ``bq_sr1`` decides accept / fallback on the device (a zero step gives
  (alpha, no u), exactly the loop's ``not np.any(s)`` branch);
* ``bq_bqnpm_metric_vk`` aggregates the slots into tau_w and a K_s-column U
  buffer with the accepted columns compacted in slot order (zero columns
  after), writes the effective rank, and computes v_k;
* the fused prox kernel reads tau_w and the effective rank from device memory
  (``bq_wtv_desc::dev_metric``): it forms the dual step from tau_w exactly as
  ``dual_step_size`` does and drops the beta warm start when the effective
  rank changed (dual_tv_solver.py:185-186).

One iteration is then two fixed launch sequences with fixed pointers: A (the
gradient, SR1, slot refresh, metric and v_k; it depends on k only through
k mod K_s) and B (the prox).  The prox kernel is specialised on the rank
(a rank-4 prox costs 1.5x a rank-1 prox at 32^3), so the host reads ONE
scalar per iteration -- the effective rank, copied to pinned memory at the
end of A -- and replays B for that rank.  Every (A, residue) and (B,
residue, rank) sequence is captured as a CUDA graph the second time it comes
up (the first run is eager; all workspaces are sized before the first
capture) and replayed afterwards.  The trace (cost, SNR, inner iterations,
elapsed device time) is recorded on the device and read once at the end --
unless an ``on_iteration`` callback is given, which needs each row as it
happens.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _abi
from . import dual_tv_solver as dts
from .fixtures import snr_db
from .metric_ops import kappa
from .tv_ops import tv_value_async

# report field offsets (bq_wtv_report): iterations int32 at 0, status int32 at 12
_REPORT_ITER = 0
_REPORT_STATUS = 3


def eligible(vs, grid, config, group) -> str:
    """'' when the resident loop applies, else the reason it does not."""
    from .physics import ScatterViewSet

    if group is not None and torch.distributed.is_initialized() and torch.distributed.get_world_size(group) > 1:
        return "view-sharded runs keep the all-reduce on the host"
    if isinstance(vs, ScatterViewSet) and vs.model == "ls":
        return "LS views: the BiCGSTAB iteration count is data dependent (host early exit)"
    if not 2 <= config.subsets <= 8:
        return "K_s outside 2..8"
    if grid.ndim != 3:
        return "the fused prox kernel is 3-D"
    k1 = grid.dims[0]
    if not ((4 <= k1 <= 128 and k1 % 4 == 0 and 128 % k1 == 0) or k1 == 256):
        return "row length outside the fused prox kernel's set"
    if isinstance(config.box.lower, np.ndarray) or isinstance(config.box.upper, np.ndarray):
        return "per-voxel box bounds"
    return ""


class ResidentBqnpm:
    def __init__(self, vs, views, grid, config, parts, alphas, use_graphs=True):
        self.vs, self.views, self.grid, self.cfg = vs, views, grid, config
        self.parts, self.alphas = parts, [float(a) for a in alphas]
        self.ks = config.subsets
        self.a = 1.0 if config.step is None else config.step
        self.lam = config.tv_weight
        dev, dt, n = vs.device, vs.dtype, grid.size
        self.dev, self.dt, self.n = dev, dt, n
        ks = self.ks
        self.X = torch.zeros(ks, n, dtype=dt, device=dev)
        self.G = torch.zeros(ks, n, dtype=dt, device=dev)
        self.Us = torch.zeros(ks, n, dtype=dt, device=dev)
        self.EST = torch.zeros(ks, 16, dtype=torch.float64, device=dev)
        self.meta = torch.zeros(128, dtype=torch.float64, device=dev)
        self.Uc = torch.zeros(ks, n, dtype=dt, device=dev)
        self.acc = torch.empty(n, dtype=dt, device=dev)
        self.v = torch.empty(n, dtype=dt, device=dev)
        self.s = torch.empty(n, dtype=dt, device=dev)
        self.m = torch.empty(n, dtype=dt, device=dev)
        self.ws = dts.ProxWorkspace(grid, dt, dev)
        self.lib = _abi.load_library()
        self.ctx = _abi.ctx_for(dev)
        self.stream = torch.cuda.Stream(dev)
        self.use_graphs = use_graphs
        self.graphs = {}
        self.seen = set()
        self.sized = False
        self.rank_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        self.rank_ev = torch.cuda.Event()
        lo, hi, _, _ = config.box.device_args(dt, dev)
        self.lo, self.hi = lo, hi

    # -- one iteration -------------------------------------------------------
    def _desc(self, v, rank, U, tau, reg, dev_metric):
        g, cfg, ws = self.grid, self.cfg, self.ws
        d = _abi.WtvDesc()
        d.ndim = g.ndim
        d.dtype = _abi.dtype_code(self.dt)
        d.dims[:] = g.dims3
        d.mode = cfg.mode.code
        d.rank = rank
        d.sign = 1
        d.accelerated = 1
        d.tau = tau
        d.reg = float(reg)
        d.step = (1.0 / (4.0 * g.ndim * (1.0 / tau) * reg)) if (reg > 0 and tau > 0) else (1.0 if reg > 0 else 0.0)
        d.eps = float(cfg.dual_eps)
        d.max_iter = int(cfg.dual_max_iter)
        d.newton_max_iter = int(cfg.newton_max_iter)
        d.newton_eps = float(cfg.newton_eps)
        d.lo, d.hi = self.lo, self.hi
        d.lo_arr = d.hi_arr = d.d = None
        d.U = U.data_ptr() if rank else None
        d.v = v.data_ptr()
        d.p, d.pb, d.p2 = ws.p.data_ptr(), ws.pb.data_ptr(), ws.p2.data_ptr()
        d.a, d.a2, d.x = ws.a.data_ptr(), ws.a2.data_ptr(), ws.x.data_ptr()
        d.beta = ws.beta.data_ptr()
        d.report = ws.report.data_ptr()
        d.dev_metric = dev_metric
        return d

    def _prox(self, desc):
        _abi.check(self.lib.bq_wtv_prox(self.ctx, desc, _abi.stream_ptr(self.dev)), "bqnpm prox")

    def warm_step(self, k):
        """k <= K_s: single-subset step with B = alpha I, plain TV weight (solvers.py:279-296)."""
        sigma = kappa(k, 1, self.ks)
        x = self.ws.x
        g = self.vs.subset_gradient(self._ids(sigma), x)
        alpha = self.alphas[sigma - 1]
        i = sigma - 1
        self.X[i].copy_(x)
        self.G[i].copy_(g)
        self.Us[i].zero_()
        self.EST[i].zero_()
        self.EST[i, 0] = alpha
        self.v.copy_(x - (self.a / alpha) * g)  # v = x - (a / tau) g, the reference's operation order
        # rank-0 prox; the warm start P / beta is kept in the workspace
        self._prox(self._desc(self.v, 0, None, alpha, self.a * self.lam, None))

    def _ids(self, sigma):
        return [self.views[i].view_id for i in self.parts[sigma - 1]]

    def qn_step(self, k):
        """k > K_s: one device-resident quasi-Newton iteration (solvers.py:281-312)."""
        ks = self.ks
        sigma = kappa(k, 1, ks)
        i = sigma - 1
        x = self.ws.x
        g = self.vs.subset_gradient(self._ids(sigma), x)
        if self.cfg.force_diagonal_metric:
            self.Us[i].zero_()
            self.EST[i].zero_()
            self.EST[i, 0] = self.alphas[i]
        else:
            torch.sub(x, self.X[i], out=self.s)
            torch.sub(g, self.G[i], out=self.m)
            _abi.check(self.lib.bq_sr1(self.ctx, _abi.dtype_code(self.dt), self.n, self.s.data_ptr(), self.m.data_ptr(),
                                       float(self.cfg.gamma), self.alphas[i], self.Us[i].data_ptr(),
                                       self.EST[i].data_ptr(), _abi.stream_ptr(self.dev)), "bqnpm sr1")
        self.X[i].copy_(x)
        self.G[i].copy_(g)
        order = [kappa(k, t, ks) - 1 for t in range(1, ks + 1)]
        xs = _abi.ptr_array([self.X[o] for o in order])
        gs = _abi.ptr_array([self.G[o] for o in order])
        us = _abi.ptr_array([self.Us[o] for o in order])
        es = _abi.ptr_array([self.EST[o] for o in order])
        _abi.check(self.lib.bq_bqnpm_metric_vk(self.ctx, _abi.dtype_code(self.dt), self.n, ks, xs, gs, us, es,
                                               float(self.a), self.Uc.data_ptr(), self.meta.data_ptr(),
                                               self.acc.data_ptr(), self.v.data_ptr(), _abi.stream_ptr(self.dev)),
                   "bqnpm metric / v_k")
        self.rank_host.copy_(self.meta[1:2], non_blocking=True)  # the one scalar the host reads

    def qn_prox(self, rank):
        """The prox at the effective rank (its kernel is specialised on the rank):
        the first `rank` columns of the compacted U, tau and the warm-start rule
        from the device scalars."""
        self._prox(self._desc(self.v, rank, self.Uc, 1.0, self.a * self.ks * self.lam, self.meta.data_ptr()))

    def size_workspaces(self):
        """One throwaway 1-iteration prox per rank 0..K_s on scratch buffers, so the
        lazily allocated near-list workspace of the loop's stream has its final
        size before any graph captures a pointer to it."""
        ws, v0 = dts.ProxWorkspace(self.grid, self.dt, self.dev), torch.zeros_like(self.v)
        U0 = torch.zeros_like(self.Uc)
        for r in range(self.ks + 1):
            d = self._desc(v0, r, U0, 1.0, 1.0, None)
            d.p, d.pb, d.p2 = ws.p.data_ptr(), ws.pb.data_ptr(), ws.p2.data_ptr()
            d.a, d.a2, d.x = ws.a.data_ptr(), ws.a2.data_ptr(), ws.x.data_ptr()
            d.beta, d.report = ws.beta.data_ptr(), ws.report.data_ptr()
            d.max_iter = 1
            self._prox(d)
        torch.cuda.current_stream(self.dev).synchronize()

    # -- trace on the device ---------------------------------------------------
    def record(self, k):
        vs = self.vs
        ids = [v.view_id for v in self.views]
        c = vs.costs(ids, self.ws.x).sum() / len(ids)
        if self.lam:
            c = c + self.lam * tv_value_async(self.grid, self.ws.x, self.cfg.mode)[0]
        self.cost[k] = c
        if self.gt is not None:
            self.err2[k] = torch.sum((self.ws.x.double() - self.gt) ** 2)
        if k > 0:
            self.inner[k] = self.ws.report[_REPORT_ITER * 4:_REPORT_ITER * 4 + 4].view(torch.int32)[0]
            self.status[k] = self.ws.report[_REPORT_STATUS * 4:_REPORT_STATUS * 4 + 4].view(torch.int32)[0]
        self.events[k].record()

    # -- the run ---------------------------------------------------------------
    def run(self, x0, ground_truth, on_iteration, tracer):
        cfg, ks = self.cfg, self.ks
        K = cfg.max_outer
        dev = self.dev
        self.gt = None if ground_truth is None else torch.as_tensor(np.asarray(ground_truth, dtype=float),
                                                                     device=dev)
        self.cost = torch.zeros(K + 1, dtype=torch.float64, device=dev)
        self.err2 = torch.zeros(K + 1, dtype=torch.float64, device=dev)
        self.inner = torch.zeros(K + 1, dtype=torch.int32, device=dev)
        self.status = torch.zeros(K + 1, dtype=torch.int32, device=dev)
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        start = torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream(dev)
        self.stream.wait_stream(main)
        with torch.cuda.stream(self.stream):
            start.record()
            self.ws.x.copy_(x0)
            self.ws.p.zero_()
            self.ws.beta.zero_()
            self.meta.zero_()
            self.record(0)
            if on_iteration is not None:
                self._emit(0, start, tracer, on_iteration)
            for k in range(1, K + 1):
                if k <= ks:
                    self.warm_step(k)
                else:
                    # graph A(k mod K_s): gradient, SR1, slot refresh, metric and v_k;
                    # the host reads the effective rank (one small D2H per iteration)
                    # and replays graph B(k mod K_s, rank): the rank-specialised prox.
                    # Each graph is captured the second time its key comes up (the
                    # first run is eager); cached instances replay from k = K_s + 1.
                    res = k % ks
                    self._run_graph(("pre", res), lambda: self.qn_step(k))
                    self.rank_ev.record()
                    self.rank_ev.synchronize()
                    rank = int(self.rank_host[0])
                    self._run_graph(("prox", res, rank), lambda: self.qn_prox(rank))
                self.record(k)
                if on_iteration is not None:
                    self._emit(k, start, tracer, on_iteration)
        main.wait_stream(self.stream)
        if on_iteration is None:
            torch.cuda.synchronize(dev)
            self._load_host()
            for k in range(K + 1):
                self._row(k, start, tracer)
        st = self.status.cpu().numpy()
        if np.any(st != 0):
            _abi.check(int(st[np.nonzero(st)[0][0]]), "bqnpm prox")
        return self.ws.x.clone()

    def _run_graph(self, key, fn):
        if key in self.graphs:
            self.graphs[key].replay()
            return
        if not self.use_graphs or key not in self.seen:
            self.seen.add(key)
            fn()
            return
        if not self.sized:
            self.size_workspaces()
            self.sized = True
        g = torch.cuda.CUDAGraph()
        # capture on the loop's own stream (its libbq workspace is already sized);
        # the low-level API skips torch.cuda.graph's gc / cache flush
        g.capture_begin()
        try:
            fn()
        finally:
            g.capture_end()
        self.graphs[key] = g
        g.replay()

    def _load_host(self):
        self._host = (self.cost.cpu().numpy(), self.err2.cpu().numpy(), self.inner.cpu().numpy())
        self._gnorm = float(torch.linalg.vector_norm(self.gt).item()) if self.gt is not None else None

    def _row(self, k, start, tracer):
        from .solvers import TraceRow

        cost, err2, inner = self._host
        if self.gt is not None:
            e = math.sqrt(float(err2[k]))
            snr = math.inf if e == 0.0 else 20.0 * math.log10(self._gnorm / e)
        else:
            snr = float("nan")
        tracer.grad_evals = k
        row = TraceRow(iteration=k, cost=float(cost[k]), snr_db=snr,
                       elapsed_s=start.elapsed_time(self.events[k]) * 1e-3, inner_iters=int(inner[k]),
                       grad_evals=k, full_grad_evals=0)
        tracer.trace.rows.append(row)
        if not math.isfinite(row.cost):
            raise FloatingPointError(f"bqnpm: cost diverged at iteration {k}")
        return row

    def _emit(self, k, start, tracer, on_iteration):
        self.events[k].synchronize()
        self._load_host()
        row = self._row(k, start, tracer)
        on_iteration(k, self.ws.x, row, {"metric_meta": self.meta} if k else {})


_CACHE = {}
_CACHE_MAX = 4


def for_run(vs, views, grid, config, parts, alphas, use_graphs=True):
    """A ResidentBqnpm for this problem, reused (with its captured graphs) by later
    runs with the same views, schedule, weights and Lipschitz constants -- the
    graphs hold pointers to the instance's buffers and the host constants of
    the kernels (alphas, gamma, a, lambda), so only an identical setup may reuse them."""
    key = (id(vs), grid.dims, config.subsets, config.step, config.tv_weight, config.gamma, config.mode,
           float(config.box.lower), float(config.box.upper), config.dual_eps, config.dual_max_iter,
           config.newton_eps, config.newton_max_iter, config.force_diagonal_metric,
           tuple(float(a) for a in alphas), tuple(tuple(int(i) for i in p) for p in parts),
           tuple(v.view_id for v in views), use_graphs)
    inst = _CACHE.get(key)
    if inst is None or inst.vs is not vs:
        inst = ResidentBqnpm(vs, views, grid, config, parts, alphas, use_graphs)
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        _CACHE[key] = inst
    return inst


__all__ = ["eligible", "ResidentBqnpm", "for_run"]

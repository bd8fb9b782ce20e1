"""CPU oracle (fp64 numpy) for the weighted-TV prox path.

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs as the checker
and the timed CPU baseline; never by the product package.

A restatement of the reference algorithm (paths under
``/root/reference/pkg/src/tvqn/``), written against flat Fortran-order
vectors viewed as C-order arrays of shape ``dims[::-1]``:

* stencils          tv_ops.py:107-159  (Neumann forward difference, exact adjoint, divergence)
* projection, TV    tv_ops.py:162-180
* metric            wpm.py:24-106      (W = tau I +/- U U^T, Woodbury with Cholesky)
* box / WPM Newton  wpm.py:109-253     (phi, generalised Jacobian on the strictly-inside
                                        set, best-residual iterate, Levenberg fallback)
* FGP prox          dual_tv_solver.py:119-250
* extension         W = diag(d) + sign U U^T (SURVEY 8c "diag(d) prox"): every 1/tau
                    becomes D^-1; reduces exactly to the reference when d == tau.

Pinned against the reference's own outputs: ``tests/golden/make_golden.py``
runs the reference functions on seeded inputs and ``tests/test_oracle.py``
checks this module against those vectors (and against the reference's
known-answer cases) before any GPU comparison trusts it.
"""

from __future__ import annotations

import math

import numpy as np

_LEVENBERG = 1e-8  # wpm.py:20


# ---------------------------------------------------------------------------
# stencils (tv_ops.py:107-159)
# ---------------------------------------------------------------------------
def _arr(dims, x):
    return np.asarray(x, dtype=float).reshape(tuple(reversed(dims)))


def _axis(dims, n):
    # dimension n (1-based, dims[0] fastest) is C-order axis ndim - n
    return len(dims) - n


def diff(dims, x, n):
    """Forward difference along dimension n with a zero far-boundary slice."""
    a = _arr(dims, x)
    ax = _axis(dims, n)
    out = np.zeros_like(a)
    k = a.shape[ax]
    if k > 1:
        head = [slice(None)] * a.ndim
        tail = [slice(None)] * a.ndim
        head[ax] = slice(0, k - 1)
        tail[ax] = slice(1, k)
        out[tuple(head)] = a[tuple(tail)] - a[tuple(head)]
    return out.reshape(-1)


def diff_adjoint(dims, y, n):
    """Transpose of ``diff``: out[k] = y[k-1] [k>=1] - y[k] [k<=K-2]."""
    a = _arr(dims, y)
    ax = _axis(dims, n)
    k = a.shape[ax]
    out = np.zeros_like(a)
    if k > 1:
        lead = [slice(None)] * a.ndim
        lag = [slice(None)] * a.ndim
        lead[ax] = slice(0, k - 1)
        lag[ax] = slice(1, k)
        # same rounding as the reference: (0 - y[k]) then + y[k-1]
        out[tuple(lead)] = -a[tuple(lead)]
        out[tuple(lag)] = out[tuple(lag)] + a[tuple(lead)]
    return out.reshape(-1)


def grad(dims, x):
    return np.stack([diff(dims, x, n) for n in range(1, len(dims) + 1)])


def div(dims, p):
    p = np.asarray(p, dtype=float)
    total = np.zeros(p.shape[1])
    for n in range(1, len(dims) + 1):
        total = total + diff_adjoint(dims, p[n - 1], n)
    return total


def project_dual(p, isotropic=True):
    p = np.asarray(p, dtype=float)
    if isotropic:
        nrm = np.sqrt((p * p).sum(axis=0))
        return p / np.maximum(nrm, 1.0)
    return np.clip(p, -1.0, 1.0)


def tv_value(dims, x, isotropic=True):
    g = grad(dims, x)
    if isotropic:
        return float(np.sqrt((g * g).sum(axis=0)).sum())
    return float(np.abs(g).sum())


# ---------------------------------------------------------------------------
# metric (wpm.py:24-106) + diag(d) extension
# ---------------------------------------------------------------------------
class Metric:
    """W = diag(dvec) + sign U U^T ; dvec = tau * ones for the reference metric."""

    def __init__(self, tau=None, U=None, sign=1, d=None, n=None):
        if d is None:
            if not (tau is not None and tau > 0):
                raise ValueError("tau must be positive")
        self.sign = int(sign)
        U = np.zeros((n or 0, 0)) if U is None else np.asarray(U, dtype=float)
        if U.ndim == 1:
            U = U[:, None]
        self.U = U
        self.n = U.shape[0] if U.size or n is None else n
        self.tau = None if d is None else None
        self.scalar = d is None
        self.tau = float(tau) if d is None else None
        self.d = None if d is None else np.asarray(d, dtype=float)
        r = U.shape[1]
        self.cap = None
        if r:
            if self.scalar:
                cap = np.eye(r) + self.sign * (U.T @ U) / self.tau
            else:
                cap = np.eye(r) + self.sign * (U.T @ (U / self.d[:, None]))
            self.L = np.linalg.cholesky(cap)  # raises LinAlgError when not PD
            self.cap = cap

    @property
    def rank(self):
        return self.U.shape[1]

    def dinv(self, x):
        return x / self.tau if self.scalar else x / self.d

    def min_diag(self):
        return self.tau if self.scalar else float(self.d.min())

    def apply(self, x):
        x = np.asarray(x, dtype=float)
        base = self.tau * x if self.scalar else self.d * x
        if self.rank:
            base = base + self.sign * (self.U @ (self.U.T @ x))
        return base

    def inverse(self, x):
        x = np.asarray(x, dtype=float)
        if self.scalar:
            out = x / self.tau
            if self.rank:
                c = _chol_solve(self.L, self.U.T @ x)
                out = out - self.sign * (self.U @ c) / (self.tau * self.tau)
            return out
        xd = x / self.d
        if self.rank:
            c = _chol_solve(self.L, self.U.T @ xd)
            xd = xd - self.sign * (self.U @ c) / self.d
        return xd

    def dense(self):
        w = np.diag(np.full(self.n, self.tau) if self.scalar else self.d)
        if self.rank:
            w = w + self.sign * self.U @ self.U.T
        return w


def _chol_solve(L, b):
    y = np.linalg.solve(L, b)
    return np.linalg.solve(L.T, y)


# ---------------------------------------------------------------------------
# weighted projection onto a box (wpm.py:136-253)
# ---------------------------------------------------------------------------
def clamp(x, lo, hi):
    return np.minimum(np.maximum(x, lo), hi)


def wpm_box(x, w: Metric, lo, hi, beta0=None, eps=1e-6, max_iter=50):
    """Returns (u, info) with info = {beta, iterations, residual, converged}."""
    x = np.asarray(x, dtype=float)
    r = w.rank
    if r == 0:
        return clamp(x, lo, hi), {"beta": np.zeros(0), "iterations": 0, "residual": 0.0, "converged": True}
    beta = np.zeros(r) if beta0 is None else np.array(beta0, dtype=float)
    best = (math.inf, beta)
    steps = 0
    ok = False
    while True:
        z = x - w.sign * w.dinv(w.U @ beta)
        cz = clamp(z, lo, hi)
        phi = w.U.T @ (x - cz) + beta
        res = float(np.sqrt(phi @ phi))
        if res < best[0]:
            best = (res, beta)
        if res <= eps:
            ok = True
            break
        if steps == max_iter:
            break
        inside = (z > lo) & (z < hi)
        ua = w.U[inside]
        if w.scalar:
            h = np.eye(r) + w.sign * (ua.T @ ua) / w.tau
        else:
            h = np.eye(r) + w.sign * (ua.T @ (ua / w.d[inside][:, None]))
        try:
            delta = np.linalg.solve(h, phi)
        except np.linalg.LinAlgError:
            mu = _LEVENBERG * np.abs(h).sum(axis=1).max()
            delta = np.linalg.solve(h + mu * np.eye(r), phi)
        beta = beta - delta
        steps += 1
    beta = best[1]
    u = clamp(x - w.sign * w.dinv(w.U @ beta), lo, hi)
    return u, {"beta": beta, "iterations": steps, "residual": best[0], "converged": ok}


# ---------------------------------------------------------------------------
# FGP dual solve (dual_tv_solver.py:119-250)
# ---------------------------------------------------------------------------
def fgp_prox(dims, v, w: Metric, reg, lo=0.0, hi=np.inf, isotropic=True, omega=None, p0=None,
             beta0=None, eps=1e-5, max_iter=100, accelerated=True, newton_eps=1e-6,
             newton_max_iter=50):
    """argmin_{lo<=x<=hi} 1/2||x - v||_W^2 + reg TV(x).  Returns a dict mirroring
    DualSolveReport (x, p_star, iterations, rel_change, converged,
    newton_iterations, beta_star)."""
    if eps <= 0 or max_iter < 1 or reg < 0:
        raise ValueError("bad solver arguments")
    v = np.asarray(v, dtype=float)
    nd, n = len(dims), v.size
    beta = None if beta0 is None else np.asarray(beta0, dtype=float)
    if beta is not None and beta.shape[0] != w.rank:
        beta = None
    omega = 1.0 / w.min_diag() if omega is None else omega
    newton = dict(eps=newton_eps, max_iter=newton_max_iter)

    def center(p):  # w(P) = v - reg W^-1 div(P)
        return v.copy() if reg == 0.0 else v - reg * w.inverse(div(dims, p))

    if reg == 0.0:
        x, info = wpm_box(v, w, lo, hi, beta, **newton)
        p = np.zeros((nd, n)) if p0 is None else np.asarray(p0)
        return dict(x=x, p_star=p, iterations=1, rel_change=0.0, converged=True,
                    newton_iterations=info["iterations"], beta_star=info["beta"])
    step = 1.0 / (4.0 * nd * omega * reg)
    p = np.zeros((nd, n)) if p0 is None else np.array(p0, dtype=float).reshape(nd, n)
    pbar = p.copy()
    t = 1.0
    total = 0
    rel = math.inf
    done = False
    it = 0
    for it in range(1, max_iter + 1):
        q, info = wpm_box(center(pbar), w, lo, hi, beta, **newton)
        beta = info["beta"]
        total += info["iterations"]
        pn = project_dual(pbar + step * grad(dims, q), isotropic)
        num = float(np.sqrt(((pn - p) ** 2).sum()))
        den = float(np.sqrt((p * p).sum()))
        rel = 0.0 if num == 0.0 else (num / den if den > 0.0 else math.inf)
        if rel < eps:
            p = pn
            done = True
            break
        if accelerated:
            tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
            pbar = pn + ((t - 1.0) / tn) * (pn - p)
            t = tn
        else:
            pbar = pn.copy()
        p = pn
    x, info = wpm_box(center(p), w, lo, hi, beta, **newton)
    total += info["iterations"]
    return dict(x=x, p_star=p, iterations=it, rel_change=float(rel), converged=done,
                newton_iterations=total, beta_star=info["beta"])


def primal_objective(dims, v, w: Metric, reg, x, isotropic=True):
    dlt = np.asarray(x, dtype=float) - v
    return 0.5 * float(dlt @ w.apply(dlt)) + reg * tv_value(dims, x, isotropic)


# ---------------------------------------------------------------------------
# SR1, metric aggregation, v_k, schedule (hessian_sr1.py:52-101, solvers.py:29-89)
# ---------------------------------------------------------------------------
def estimate_sr1(s, m, gamma=0.8, alpha=1.0):
    """Returns (tau, u or None)."""
    s = np.asarray(s, dtype=float)
    m = np.asarray(m, dtype=float)
    if not s.any():
        raise ValueError("degenerate step: s must be nonzero")
    if not 0.0 < gamma < 1.0 or not alpha > 0:
        raise ValueError("bad SR1 parameters")
    sm = float(s @ m)
    if sm == 0.0:
        return alpha, None
    tau = gamma * float(m @ m) / sm
    if tau < 0.0:
        return alpha, None
    res = m - tau * s
    curv = float(res @ s)
    if curv <= 1e-8 * np.sqrt(s @ s) * np.sqrt(res @ res) or curv <= 0.0:
        return tau, None
    u = res / math.sqrt(curv)
    return tau, (u if u.any() else None)


def kappa(k, t, ks):
    if not 1 <= t <= ks:
        raise ValueError("term index out of range")
    return (k - 1 - t) % ks + 1


def partition_views(n_views, n_subsets, strategy="equispaced"):
    if not 1 <= n_subsets <= n_views:
        raise ValueError("bad subset count")
    idx = np.arange(n_views)
    if strategy == "equispaced":
        return [idx[t::n_subsets] for t in range(n_subsets)]
    if strategy == "contiguous":
        return list(np.array_split(idx, n_subsets))
    raise ValueError(strategy)


def aggregate(slots):
    """slots: list of (x, g, tau, u|None) -> Metric(sum tau, nonzero u columns)."""
    tau = sum(sl[2] for sl in slots)
    cols = [sl[3] for sl in slots if sl[3] is not None]
    n = slots[0][0].shape[0]
    U = np.column_stack(cols) if cols else np.zeros((n, 0))
    return Metric(tau=tau, U=U)


def v_k(slots, w: Metric, step):
    acc = np.zeros_like(slots[0][0])
    for x, g, tau, u in slots:
        bx = tau * x
        if u is not None:
            bx = bx + u * float(u @ x)
        acc = acc + (bx - step * g)
    return w.inverse(acc)

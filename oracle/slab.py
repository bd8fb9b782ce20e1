"""Numpy backend of the z-slab prox passes -- TEST INFRASTRUCTURE ONLY.

Plugs into ``paper_2307_02043_b200.slab_prox.slab_solve`` in place of the
device backend so the sharded control code (halo exchange, all-reduces,
replicated Newton / FGP decisions) is checked on CPU with gloo at world size
2 against the unsharded oracle ``oracle.prox.fgp_prox`` (which follows
dual_tv_solver.py:161-250).  Each pass restates one ``csrc/slab_prox.cu``
kernel on a slab of planes [z0, z1) of a (K1, K2, K3) grid, flat Fortran
order (x fastest); the per-voxel arithmetic is that of oracle/prox.py.
"""

from __future__ import annotations

import numpy as np
import torch


class NumpySlabs:
    def __init__(self, dims, bounds, k3, v, U, d=None, *, rank, sign, tau, reg, lo, hi, iso=True):
        self.K1, self.K2 = int(dims[0]), int(dims[1])
        self.plane = self.K1 * self.K2
        self.bounds, self.k3 = list(bounds), int(k3)
        pl = self.plane
        self.v = [np.asarray(v[z0 * pl:z1 * pl], float) for z0, z1 in bounds]
        self.U = [np.asarray(U[z0 * pl:z1 * pl], float).reshape(-1, rank) if rank else None for z0, z1 in bounds]
        self.d = [np.asarray(d[z0 * pl:z1 * pl], float) if d is not None else None for z0, z1 in bounds]
        self.rank, self.sign, self.tau, self.reg = rank, sign, tau, reg
        self.lo, self.hi, self.iso = lo, hi, iso
        self.cb = {}

    # ---- helpers -------------------------------------------------------------
    def _L(self, s):
        z0, z1 = self.bounds[s]
        return z1 - z0

    def _dinv(self, s, x):
        return x / self.d[s] if self.d[s] is not None else x / self.tau

    def _center(self, s, t, c):
        if self.rank:
            return self.v[s] - self.reg * (t - self.sign * self._dinv(s, self.U[s] @ c))
        return self.v[s] - self.reg * t

    def _z(self, s, w, beta):
        if not self.rank:
            return w
        return w - self.sign * self._dinv(s, self.U[s] @ beta)

    # ---- the backend interface of slab_prox.slab_solve -------------------------
    def zeros(self, s):
        return torch.zeros(self._L(s) * self.plane, dtype=torch.float64)

    def dual_field(self, s, init):
        n = self._L(s) * self.plane
        return torch.zeros(3, n, dtype=torch.float64) if init is None else torch.as_tensor(init).reshape(3, n).clone()

    def top_plane_z(self, field):
        return field[2, -self.plane:].clone()

    def bottom_plane(self, q):
        return q[: self.plane].clone()

    def div(self, s, field, halo):
        z0, z1 = self.bounds[s]
        L = z1 - z0
        F = field.numpy().reshape(3, L, self.K2, self.K1)
        out = np.zeros((L, self.K2, self.K1))
        for a, ax in ((0, 2), (1, 1)):  # x then y: out[k] += y[k-1] - y[k] inside (tv_ops.py:129-131)
            y = F[a]
            o = np.zeros_like(y)
            sl = [slice(None)] * 3
            sl[ax] = slice(None, -1)
            o[tuple(sl)] -= y[tuple(sl)]
            sl2 = [slice(None)] * 3
            sl2[ax] = slice(1, None)
            o[tuple(sl2)] += y[tuple(sl)]
            out += o
        y = F[2]
        o = np.zeros_like(y)
        last = L if z1 < self.k3 else L - 1  # the global last plane has no forward difference
        o[:last] -= y[:last]
        o[1:] += y[:-1]
        if z0 > 0:
            o[0] += halo.numpy().reshape(self.K2, self.K1)
        out += o
        t = self._dinv(s, out.reshape(-1))
        sv = self.U[s].T @ t if self.rank else np.zeros(0)
        return torch.from_numpy(t), torch.from_numpy(np.asarray(sv, float))

    # ---- control block: the numpy statement of bq_slab_ctl (csrc/slab_prox.cu) ----
    def ctl(self, op, inp, newton_eps, newton_max_iter, eps):
        r = self.rank
        c = self.cb
        a = None if inp is None else (inp.numpy() if isinstance(inp, torch.Tensor) else np.asarray(inp, float))
        if op == 0:
            c.update(L=a[: r * r].reshape(r, r) if r else None, beta=a[64:64 + r].copy(), total=0, fgp=0,
                     rel=np.inf, done=r == 0)
        elif op == 1:
            c["coef"] = np.linalg.solve(c["L"].T, np.linalg.solve(c["L"], a[:r])) if r else np.zeros(0)
            c.update(saved=c["beta"].copy(), best_beta=c["beta"].copy(), best=np.inf, it=0, last=0, done=r == 0)
        elif op == 2:
            if c["done"]:
                return
            res_vec = a[:r] + c["beta"]
            res = float(np.linalg.norm(res_vec))
            if res < c["best"]:
                c["best"], c["best_beta"] = res, c["beta"].copy()
            if res <= newton_eps or c["it"] == newton_max_iter:
                c["beta"] = c["best_beta"].copy()
                c["last"] = c["it"]
                c["total"] += c["it"]
                c["done"] = True
                return
            g = np.zeros((r, r))
            k = r
            for i in range(r):
                for j in range(i + 1):
                    g[i, j] = g[j, i] = a[k]
                    k += 1
            h = np.eye(r) + self.sign * (g / self.tau if self.d[0] is None else g)
            try:
                step = np.linalg.solve(h, res_vec)
            except np.linalg.LinAlgError:
                mu = 1e-8 * np.linalg.norm(h, np.inf)
                step = np.linalg.solve(h + mu * np.eye(r), res_vec)
            c["beta"] = c["beta"] - step
            c["it"] += 1
        elif op == 3:
            num, den = np.sqrt(a[0]), np.sqrt(a[1])
            c["rel"] = 0.0 if num == 0.0 else (num / den if den > 0.0 else np.inf)
            c["fgp"] = c["rel"] < eps
        elif op == 4:
            c["beta"] = c["saved"].copy()
            if c["done"]:
                c["total"] -= c["last"]

    def read_ctl(self):
        c = self.cb
        out = np.zeros(128)
        out[0], out[1], out[3], out[4], out[5], out[6] = c["done"], c["it"], c["total"], c["rel"], c["fgp"], c["last"]
        out[8:8 + self.rank] = c["beta"]
        return out

    def newton(self, s, t):
        t = t.numpy()
        w = self._center(s, t, self.cb["coef"])
        z = self._z(s, w, self.cb["beta"])
        q = np.clip(z, self.lo, self.hi)
        U = self.U[s]
        phi = U.T @ (w - q)
        ins = (z > self.lo) & (z < self.hi)
        ua = U[ins]
        g = ua.T @ (ua / self.d[s][ins][:, None]) if self.d[s] is not None else ua.T @ ua
        tri = [g[i, j] for i in range(self.rank) for j in range(i + 1)]
        return torch.from_numpy(np.concatenate([phi, tri]))

    def q(self, s, t):
        w = self._center(s, t.numpy(), self.cb["coef"])
        return torch.from_numpy(np.clip(self._z(s, w, self.cb["beta"]), self.lo, self.hi))

    def dual(self, s, pbar, p, q, halo, step, mom):
        z0, z1 = self.bounds[s]
        L = z1 - z0
        qv = q.numpy().reshape(L, self.K2, self.K1)
        g = np.zeros((3, L, self.K2, self.K1))
        g[0, :, :, :-1] = qv[:, :, 1:] - qv[:, :, :-1]
        g[1, :, :-1, :] = qv[:, 1:, :] - qv[:, :-1, :]
        g[2, :-1] = qv[1:] - qv[:-1]
        if z1 < self.k3:
            g[2, -1] = halo.numpy().reshape(self.K2, self.K1) - qv[-1]
        w = pbar.numpy() + step * g.reshape(3, -1)
        if self.iso:
            w = w / np.maximum(np.sqrt(np.sum(w * w, axis=0)), 1.0)
        else:
            w = np.clip(w, -1.0, 1.0)
        pv = p.numpy()
        dl = w - pv
        norms = np.array([float(np.sum(dl * dl)), float(np.sum(pv * pv))])
        return torch.from_numpy(w), torch.from_numpy(w + mom * dl), torch.from_numpy(norms)

    def concat(self, parts):
        return torch.cat(parts)

    def concat_dual(self, parts):
        return torch.cat(parts, dim=1)

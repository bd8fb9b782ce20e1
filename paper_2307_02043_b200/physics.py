"""First-Born and Lippmann-Schwinger view batches on the device (north star (1)(2)).

No reference implementation exists; the
discretisation is specified once in ``oracle/physics.py`` (Green's kernel on
the 2n-padded grid with a ball-averaged self term, plane-wave incidence,
detector one voxel past the +z face, BiCGSTAB from x0 = 0 with a relative
residual tolerance) and implemented here on libbq:

* ``bq_green_init``  : FFT of the Green kernel, once per setup
* ``bq_ls_conv``     : padded Green convolution as five pruned line passes
                       (ls_fft.cu; cuFFT on the padded grid for other sizes)
* ``bq_ls_bicgstab`` : batched BiCGSTAB run on the device (per-view scalars and
                       stopping tests on the GPU, dots fused into the producing
                       kernels, converged views skipped)
* ``bq_ls_grad_accum`` : Re(conj(f' u) . w) summed over the views of the batch

The views plug into the reference's ``ViewProblem`` contract
(forward_models.py:25-83) with real-packed [Re; Im] detector data,
and ``subset_gradient`` batches a whole subset.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _abi
from ._tensors import default_device, is_torch, out_like, to_dev


class ScatterViewSet:
    """L plane-wave views of an n^3 grid (model 'born' or 'ls')."""

    def __init__(self, n, n_views, model="ls", h=0.1, lam0=0.406, n_b=1.333, theta_deg=35.0,
                 dtype=torch.complex64, tol=1e-6, max_iter=500, batch=8, device=None):
        if model not in ("born", "ls"):
            raise ValueError(f"unknown model {model!r}")
        if dtype not in (torch.complex64, torch.complex128):
            raise ValueError("dtype must be complex64 or complex128")
        self.n, self.L, self.model = int(n), int(n_views), model
        self.h, self.lam0, self.n_b, self.theta = float(h), float(lam0), float(n_b), float(theta_deg)
        self.k0 = 2.0 * math.pi / self.lam0
        self.kb = self.n_b * self.k0
        self.cdtype = dtype
        self.rdtype = torch.float32 if dtype == torch.complex64 else torch.float64
        self.code = _abi.BQ_F32 if dtype == torch.complex64 else _abi.BQ_F64
        self.tol, self.max_iter, self.batch = float(tol), int(max_iter), int(batch)
        self.device = device or default_device()
        self.N = self.n ** 3
        self.lib = _abi.load_library()
        self.ctx = _abi.ctx_for(self.device)
        m = 2 * self.n
        self.khat = torch.empty(m, m, m, dtype=dtype, device=self.device)
        self._check(self.lib.bq_green_init(self.ctx, self.code, self.n, self.h, self.kb, self.khat.data_ptr(),
                                           self._st()), "green_init")
        th = math.radians(self.theta)
        kv = []
        for l in range(self.L):
            ph = 2.0 * math.pi * l / self.L
            kv.append([self.kb * math.sin(th) * math.cos(ph), self.kb * math.sin(th) * math.sin(ph),
                       self.kb * math.cos(th)])
        self.kvec = torch.tensor(kv, dtype=torch.float64, device=self.device)
        self.y = torch.zeros(self.L, 2 * self.n * self.n, dtype=self.rdtype, device=self.device)
        self._pad = {}
        self.iters_forward = []
        self.iters_adjoint = []

    @property
    def dtype(self):
        """Real field dtype of x and of the gradient (the solver loop's working type)."""
        return self.rdtype

    # -- plumbing ---------------------------------------------------------------
    def _st(self):
        return _abi.stream_ptr(self.device)

    def _check(self, rc, what):
        _abi.check(rc, what)

    def _padbuf(self, B):
        if B not in self._pad:
            m = 2 * self.n
            self._pad[B] = torch.empty(B, m, m, m, dtype=self.cdtype, device=self.device)
        return self._pad[B]

    def potential(self, x):
        f = torch.empty(self.N, dtype=self.rdtype, device=self.device)
        fp = torch.empty_like(f)
        self._check(self.lib.bq_ls_potential(self.ctx, self.code, self.N, x.data_ptr(), self.k0, self.n_b,
                                             int(self.model == "born"), f.data_ptr(), fp.data_ptr(), self._st()),
                    "potential")
        return f, fp

    def _index(self, views):
        """Device index of a view batch, cached (no host-to-device copy per call,
        so a Born subset gradient can be captured in a CUDA graph)."""
        key = tuple(int(v) for v in views)
        cache = self.__dict__.setdefault("_idx_cache", {})
        if key not in cache:
            cache[key] = torch.tensor(key, dtype=torch.long, device=self.device)
        return cache[key]

    def _rows(self, t, views):
        return t.index_select(0, self._index(views))

    def incident(self, views):
        B = len(views)
        kv = self._rows(self.kvec, views).contiguous()
        out = torch.empty(B, self.N, dtype=self.cdtype, device=self.device)
        self._check(self.lib.bq_ls_incident(self.ctx, self.code, self.n, self.h, B, kv.data_ptr(), out.data_ptr(),
                                            self._st()), "incident")
        return out

    def conv(self, op, f, v, alpha=0.0, beta=1.0, addend=None):
        B = v.shape[0]
        out_len = self.n * self.n if op == 2 else self.N
        out = torch.empty(B, out_len, dtype=self.cdtype, device=self.device)
        self._check(self.lib.bq_ls_conv(self.ctx, self.code, self.n, B, op, self.khat.data_ptr(), _abi.ptr(f),
                                        v.data_ptr(), float(alpha), float(beta), _abi.ptr(addend),
                                        self._padbuf(B).data_ptr(), out.data_ptr(), self._st()), "ls_conv")
        return out

    # -- batched BiCGSTAB (oracle/physics.py bicgstab) ------------------------
    def solve(self, adjoint, f, b):
        """x_b = A^-1 b_b for the B views of `b` (adjoint: A^H), BiCGSTAB from x0 = 0 to
        the relative residual `tol`, run entirely on the device (bq_ls_bicgstab:
        scalar recurrences and stopping tests on the GPU, converged views skipped).
        Returns (x, iterations per view)."""
        B, N = b.shape
        key = (B, "bicg")
        if key not in self._pad:
            small = int(self.lib.bq_ls_bicgstab_small_bytes(self.ctx, self.n, B))
            if small < 0:
                raise ValueError("bq_ls_bicgstab_small_bytes failed")
            self._pad[key] = (torch.empty(6, B, N, dtype=self.cdtype, device=self.device),
                              torch.empty(small, dtype=torch.uint8, device=self.device),
                              torch.empty(B, dtype=torch.int32, device=self.device))
        vec, small, iters = self._pad[key]
        b = b.contiguous()
        x = torch.empty_like(b)
        self._check(self.lib.bq_ls_bicgstab(self.ctx, self.code, self.n, B, int(adjoint), self.khat.data_ptr(),
                                            f.data_ptr(), b.data_ptr(), x.data_ptr(), self.tol, self.max_iter,
                                            vec.data_ptr(), self._padbuf(B).data_ptr(), small.data_ptr(),
                                            iters.data_ptr(), self._st()), "ls_bicgstab")
        return x, iters.cpu().numpy().astype(np.int64)

    # -- operators ---------------------------------------------------------------
    # -- operators ---------------------------------------------------------------
    def total_field(self, f, views):
        uin = self.incident(views)
        if self.model == "born":
            return uin, np.zeros(len(views), dtype=np.int64)
        return self.solve(False, f, uin)

    def forward_c(self, x, views):
        f, _ = self.potential(x)
        u, it = self.total_field(f, views)
        self.iters_forward.extend(int(i) for i in it)
        return self.conv(2, f, u)

    @staticmethod
    def pack(dc):
        return torch.cat([dc.real, dc.imag], dim=1)

    def unpack(self, rr):
        nn = self.n * self.n
        return torch.complex(rr[:, :nn].contiguous(), rr[:, nn:].contiguous()).to(self.cdtype)

    def forward(self, x, views):
        return self.pack(self.forward_c(x, views))

    def vjp_from_residual(self, x, views, r_c, f, fp, u, grad, scale, accumulate):
        w = self.conv(3, None, r_c)
        if self.model == "ls":
            z, it = self.solve(True, f, self._cmul_conj_f(f, w))
            self.iters_adjoint.extend(int(i) for i in it)
            w = self.conv(1, None, z, 0.0, 1.0, addend=w)  # w + G_dom^H z
        self._check(self.lib.bq_ls_grad_accum(self.ctx, self.code, self.N, len(views), fp.data_ptr(), u.data_ptr(),
                                              w.contiguous().data_ptr(), float(scale), grad.data_ptr(),
                                              int(accumulate), self._st()), "grad_accum")
        return grad

    def _cmul_conj_f(self, f, w):
        # conj(f) . w with real f: a real scaling of each view
        out = torch.empty_like(w)
        self._check(self.lib.bq_cscale_real(self.ctx, self.code, self.N, w.shape[0], f.data_ptr(), w.data_ptr(),
                                            out.data_ptr(), self._st()), "cscale")
        return out

    def subset_gradient(self, views, x):
        """(1/|S|) sum_rho grad 1/2 ||H_rho(x) - y_rho||^2, views batched `batch` at a time."""
        views = list(views)
        grad = torch.zeros(self.N, dtype=self.rdtype, device=self.device)
        f, fp = self.potential(x)
        first = True
        for i in range(0, len(views), self.batch):
            vb = views[i:i + self.batch]
            u, it = self.total_field(f, vb)
            self.iters_forward.extend(int(k) for k in it)
            H = self.conv(2, f, u)
            r = H - self.unpack(self._rows(self.y, vb))
            self.vjp_from_residual(x, vb, r, f, fp, u, grad, 1.0 / len(views), accumulate=not first)
            first = False
        return grad

    def jvp(self, views, x, dx, f=None, fp=None, u=None):
        """J_rho dx for the views of a batch (complex detector data)."""
        if f is None:
            f, fp = self.potential(x)
        if u is None:
            u, _ = self.total_field(f, views)
        # q = f' u dx  (dx real, one N-vector shared by the batch)
        q = torch.empty_like(u)
        fpdx = torch.empty_like(f)
        self._check(self.lib.bq_pointwise(self.ctx, self.code, 2, self.N, None, fp.data_ptr(), dx.data_ptr(), 0.0,
                                          fpdx.data_ptr(), self._st()), "pointwise")
        self._check(self.lib.bq_cscale_real(self.ctx, self.code, self.N, u.shape[0], fpdx.data_ptr(), u.data_ptr(),
                                            q.data_ptr(), self._st()), "cscale")
        if self.model == "ls":
            rhs = self.conv(0, None, q)  # G_dom q
            z, _ = self.solve(False, f, rhs)
            fz = self._cmul_conj_f(f, z)  # f real: f . z
            q = q + fz
        return self.conv(2, None, q)

    def gauss_newton_subset(self, views, x, v):
        """(1/|S|) sum_rho J_rho^T J_rho v (solvers.py:176-181), batched."""
        views = list(views)
        out = torch.zeros(self.N, dtype=self.rdtype, device=self.device)
        f, fp = self.potential(x)
        first = True
        for i in range(0, len(views), self.batch):
            vb = views[i:i + self.batch]
            u, _ = self.total_field(f, vb)
            jv = self.jvp(vb, x, v, f, fp, u)
            self.vjp_from_residual(x, vb, jv, f, fp, u, out, 1.0 / len(views), accumulate=not first)
            first = False
        return out

    def mean_adjoint_measurements(self, views):
        """(1/L) sum_rho J_rho(0)^T y_rho (solvers.py:192-199)."""
        views = list(views)
        x0 = torch.zeros(self.N, dtype=self.rdtype, device=self.device)
        out = torch.zeros_like(x0)
        f, fp = self.potential(x0)
        first = True
        for i in range(0, len(views), self.batch):
            vb = views[i:i + self.batch]
            u = self.incident(vb)  # f = 0: the total field is the incident one
            self.vjp_from_residual(x0, vb, self.unpack(self._rows(self.y, vb)), f, fp, u, out, 1.0 / len(views),
                                   accumulate=not first)
            first = False
        return out

    def costs(self, views, x):
        views = list(views)
        out = []
        for i in range(0, len(views), self.batch):
            vb = views[i:i + self.batch]
            d = self.forward(x, vb) - self._rows(self.y, vb)
            out.append(0.5 * (d.double() ** 2).sum(dim=1))
        return torch.cat(out)


class ScatterView:
    """ViewProblem-compatible single view (forward_models.py:25-83)."""

    def __init__(self, vs: ScatterViewSet, v: int):
        self.viewset, self.view_id = vs, int(v)

    @property
    def y(self):
        return self.viewset.y[self.view_id].detach().cpu().numpy().astype(float)

    def _x(self, x):
        return to_dev(x, self.viewset.rdtype, self.viewset.device)

    def forward(self, x):
        return out_like(x, self.viewset.forward(self._x(x), [self.view_id])[0])

    def gradient(self, x):
        return out_like(x, self.viewset.subset_gradient([self.view_id], self._x(x)))

    def value(self, x):
        return float(self.viewset.costs([self.view_id], self._x(x))[0].item())

    def jacobian_vec(self, x, v):
        """J(x) v as real-packed [Re; Im] detector data (the JVP of ``forward``)."""
        vs = self.viewset
        xt = self._x(x)
        vt = to_dev(v, vs.rdtype, vs.device).reshape(-1)
        return out_like(v, vs.pack(vs.jvp([self.view_id], xt, vt))[0])

    def self_check(self, n, rng, adj_tol=1e-10, grad_tol=1e-4, x_scale=0.02):
        """The reference's plugin check (forward_models.py:66-83): adjoint identity
        <J v, z> = <v, J^T z> and a central finite-difference gradient test,
        same draw order from `rng` (x, v, z, then the direction).  Raises
        RuntimeError on failure.

        Differences, both forced by the physics: x is the drawn normal vector
        times `x_scale` (x is a refractive-index contrast, O(0.01-0.1); a unit
        contrast makes the Lippmann-Schwinger series diverge), and a complex64
        view set checks at its own precision (adjoint >= 1e-4, gradient >= 1e-2,
        h = 1e-3) instead of the fp64 tolerances."""
        vs = self.viewset
        x = rng.standard_normal(n) * x_scale
        v = rng.standard_normal(n)
        z = rng.standard_normal(2 * vs.n * vs.n)
        single = vs.cdtype == torch.complex64
        adj_tol = max(adj_tol, 1e-4) if single else adj_tol
        grad_tol = max(grad_tol, 1e-2) if single else grad_tol
        lhs = float(np.dot(self.jacobian_vec(x, v), z))
        rhs = float(np.dot(v, self.adjoint_vec(x, z)))
        if abs(lhs - rhs) > adj_tol * max(1.0, abs(lhs), abs(rhs)):
            raise RuntimeError(f"view {self.view_id}: adjoint test failed ({lhs} vs {rhs})")
        g = self.gradient(x)
        h = 1e-3 * x_scale if single else 1e-6 * x_scale
        d = rng.standard_normal(n)
        d /= np.linalg.norm(d)
        fd = (self.value(x + h * d) - self.value(x - h * d)) / (2 * h)
        an = float(np.dot(g, d))
        if abs(fd - an) > grad_tol * max(1.0, abs(fd), abs(an)):
            raise RuntimeError(f"view {self.view_id}: gradient test failed ({an} vs {fd})")

    def adjoint_vec(self, x, z):
        vs = self.viewset
        xt = self._x(x)
        f, fp = vs.potential(xt)
        u, _ = vs.total_field(f, [self.view_id])
        zt = to_dev(z, vs.rdtype, vs.device)[None, :]
        grad = torch.zeros(vs.N, dtype=vs.rdtype, device=vs.device)
        vs.vjp_from_residual(xt, [self.view_id], vs.unpack(zt), f, fp, u, grad, 1.0, accumulate=False)
        return out_like(z, grad)


def make_scatter_views(n, n_views, model="ls", x_gt=None, noise_snr_db=None, seed=0, self_check=False, **kw):
    """Views with synthetic measurements y = H(x_gt) (+ complex Gaussian noise at
    the given SNR, 20 log10(||y|| / ||e||), as forward_models.py:186-191).
    ``self_check`` runs every view's ``ViewProblem.self_check`` after the data is
    drawn, as the reference's view factory does (forward_models.py:193); off by
    default because at n = 128 each check is several LS solves."""
    vs = ScatterViewSet(n, n_views, model=model, **kw)
    rng = np.random.default_rng(seed)
    if x_gt is not None:
        xt = to_dev(x_gt, vs.rdtype, vs.device)
        for i in range(0, n_views, vs.batch):
            vb = list(range(i, min(n_views, i + vs.batch)))
            vs.y[vb] = vs.forward(xt, vb)
        if noise_snr_db is not None:
            for l in range(n_views):
                e = rng.standard_normal(vs.y.shape[1])
                scale = float(torch.linalg.vector_norm(vs.y[l].double()).item()) / np.linalg.norm(e)
                vs.y[l] += to_dev(e * scale * 10.0 ** (-noise_snr_db / 20.0), vs.rdtype, vs.device)
    views = [ScatterView(vs, l) for l in range(n_views)]
    if self_check:
        for view in views:
            view.self_check(vs.N, rng)
    return views, vs


__all__ = ["ScatterViewSet", "ScatterView", "make_scatter_views"]

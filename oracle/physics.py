"""CPU oracle (complex128 numpy) for the first-Born and Lippmann-Schwinger views.

TEST INFRASTRUCTURE ONLY.  PARITY UNPINNED: the reference package contains no
Born/LS physics (PAPER.md:614 defers H_rho to a
supplementary that is not in the container).  This module is the builder's
specification of the discretisation (decision D-2),
implemented once here and once on the device.  Trust comes from properties
(tests/test_physics_oracle.py): adjointness, finite-difference gradients, the
Born limit as the contrast -> 0, reciprocity, zero fidelity at the truth, and
the reference's ViewProblem contract (forward_models.py:25-83).

Specification
-------------
* Grid n^3 voxels of side h, voxel centres r_j = h (j + 1/2).  Unknown x = Delta n
  >= 0 (refractive-index contrast), background n_b, k0 = 2 pi / lambda0,
  k_b = n_b k0.
* Scattering potential f(x) = k0^2 ((n_b + x)^2 - n_b^2) (LS); the convex first-Born
  model uses the linearisation f = 2 k0^2 n_b x (decision D-1).
* Incident plane wave of view l: u_in(r) = exp(i k_l . r),
  k_l = k_b (sin th cos ph_l, sin th sin ph_l, cos th), ph_l = 2 pi l / L.
* Green's operator: (G v)(r_t) = sum_j K(r_t - r_j) v_j with
  K(d) = h^3 exp(i k_b |d|) / (4 pi |d|) for d != 0 and the ball-averaged self term
  K(0) = (exp(i k_b a)(1 - i k_b a) - 1) / k_b^2, a = h (3 / (4 pi))^(1/3).
  Evaluated as an exact aperiodic convolution on the 2n-padded grid: offsets
  represented as i (i <= n) or i - 2n (i > n), so every target in planes 0..n
  and every source in 0..n-1 is aliasing-free.
* LS: solve (I - G_dom diag f) u = u_in on the domain (BiCGSTAB, x0 = 0,
  relative residual tol), detector = scattered field on plane z = n (one voxel
  past the +z face): H(x) = P_det G (f u), an n^2 complex vector, packed as real
  [Re; Im].
* Born: u = u_in (no solve).
* Gradient of 1/2 ||H(x) - y||^2: with A = I - G_dom diag f,
  J dx = P_det G (I + diag(f) A^-1 G_dom) diag(f'(x) u) dx  and
  grad = Re( conj(f' u) . (w + G_dom^H A^-H (conj(f) . w)) ),  w = G^H P_det^T r.
  (Born: grad = Re(conj(f' u_in) . w).)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import os

import numpy as np
import scipy.fft as _sfft

# all host cores for the padded transforms (scipy's pocketfft; the result
# differs from numpy.fft only by rounding)
_W = int(os.environ.get("BQ_ORACLE_FFT_WORKERS", "0")) or (os.cpu_count() or 1)


def _fftn(a):
    return _sfft.fftn(a, workers=_W)


def _ifftn(a):
    return _sfft.ifftn(a, workers=_W)


@dataclass(frozen=True)
class Setup:
    n: int
    h: float = 0.1        # um
    lam0: float = 0.406   # um
    n_b: float = 1.333
    theta_deg: float = 35.0
    n_views: int = 16

    @property
    def k0(self):
        return 2.0 * math.pi / self.lam0

    @property
    def kb(self):
        return self.n_b * self.k0


def green_kernel_hat(s: Setup, dtype=np.complex128):
    """FFT of the offset kernel K on the (2n)^3 padded grid (C order: z, y, x)."""
    n, m = s.n, 2 * s.n
    off = np.arange(m, dtype=float)
    off = np.where(off <= n, off, off - m) * s.h
    dz, dy, dx = np.meshgrid(off, off, off, indexing="ij")
    r = np.sqrt(dx * dx + dy * dy + dz * dz)
    kb = s.kb
    with np.errstate(divide="ignore", invalid="ignore"):
        K = s.h ** 3 * np.exp(1j * kb * r) / (4.0 * math.pi * r)
    a = s.h * (3.0 / (4.0 * math.pi)) ** (1.0 / 3.0)
    K[0, 0, 0] = (np.exp(1j * kb * a) * (1.0 - 1j * kb * a) - 1.0) / kb ** 2
    return _fftn(K).astype(dtype)


def incident(s: Setup, view: int):
    n = s.n
    ph = 2.0 * math.pi * view / s.n_views
    th = math.radians(s.theta_deg)
    kx, ky, kz = s.kb * math.sin(th) * math.cos(ph), s.kb * math.sin(th) * math.sin(ph), s.kb * math.cos(th)
    c = (np.arange(n) + 0.5) * s.h
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return np.exp(1j * (kx * x + ky * y + kz * z))  # C order (z, y, x) == flat Fortran over (x, y, z)


class Green:
    def __init__(self, s: Setup):
        self.s = s
        self.Kh = green_kernel_hat(s)

    def _pad(self, v):
        n = self.s.n
        buf = np.zeros((2 * n,) * 3, dtype=complex)
        buf[:n, :n, :n] = v.reshape(n, n, n)
        return buf

    def apply_full(self, v):
        """G v on the padded grid (targets anywhere in planes 0..n)."""
        return _ifftn(self.Kh * _fftn(self._pad(v)))

    def dom(self, v):
        n = self.s.n
        return self.apply_full(v)[:n, :n, :n].reshape(-1)

    def det(self, v):
        n = self.s.n
        return self.apply_full(v)[n, :n, :n].reshape(-1)

    def _adj_from_padded(self, buf):
        n = self.s.n
        return _ifftn(np.conj(self.Kh) * _fftn(buf))[:n, :n, :n].reshape(-1)

    def dom_adj(self, w):
        return self._adj_from_padded(self._pad(w))

    def det_adj(self, r):
        n = self.s.n
        buf = np.zeros((2 * n,) * 3, dtype=complex)
        buf[n, :n, :n] = r.reshape(n, n)
        return self._adj_from_padded(buf)


def bicgstab(apply_a, b, tol=1e-6, max_iter=500, x0=None):
    """Unpreconditioned BiCGSTAB (van der Vorst); relative residual ||r|| <= tol ||b||.
    Returns (x, iterations, rel_residual).  <a, b> = sum conj(a) b."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - apply_a(x) if x0 is not None else b.copy()
    rh = r.copy()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return x, 0, 0.0
    rho = alpha = omega = 1.0 + 0.0j
    v = np.zeros_like(b)
    p = np.zeros_like(b)
    it = 0
    res = np.linalg.norm(r) / nb
    if res <= tol:
        return x, 0, res
    for it in range(1, max_iter + 1):
        rho_new = np.vdot(rh, r)
        beta = (rho_new / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        v = apply_a(p)
        alpha = rho_new / np.vdot(rh, v)
        s = r - alpha * v
        if np.linalg.norm(s) <= tol * nb:
            x = x + alpha * p
            res = np.linalg.norm(s) / nb
            break
        t = apply_a(s)
        omega = np.vdot(t, s) / np.vdot(t, t)
        x = x + alpha * p + omega * s
        r = s - omega * t
        rho = rho_new
        res = np.linalg.norm(r) / nb
        if res <= tol:
            break
    return x, it, res


class ScatterModel:
    """Born / LS measurement maps for one setup."""

    def __init__(self, s: Setup, model="ls", tol=1e-6, max_iter=500):
        if model not in ("born", "ls"):
            raise ValueError(model)
        self.s, self.model, self.tol, self.max_iter = s, model, tol, max_iter
        self.G = Green(s)
        self.last_iters = []

    def pot(self, x):
        k0, nb = self.s.k0, self.s.n_b
        x = np.asarray(x, dtype=float)
        if self.model == "born":
            return 2.0 * k0 * k0 * nb * x, np.full_like(x, 2.0 * k0 * k0 * nb)
        return k0 * k0 * ((nb + x) ** 2 - nb * nb), 2.0 * k0 * k0 * (nb + x)

    def total_field(self, x, view):
        uin = incident(self.s, view).reshape(-1)
        if self.model == "born":
            return uin, 0
        f, _ = self.pot(x)
        u, it, _ = bicgstab(lambda v: v - self.G.dom(f * v), uin, self.tol, self.max_iter)
        return u, it

    def forward_c(self, x, view):
        f, _ = self.pot(x)
        u, it = self.total_field(x, view)
        self.last_iters.append(it)
        return self.G.det(f * u)

    def forward(self, x, view):
        d = self.forward_c(x, view)
        return np.concatenate([d.real, d.imag])

    def jvp(self, x, view, dx):
        f, fp = self.pot(x)
        u, _ = self.total_field(x, view)
        q = fp * u * dx
        if self.model == "ls":
            z, _, _ = bicgstab(lambda v: v - self.G.dom(f * v), self.G.dom(q), self.tol, self.max_iter)
            q = q + f * z
        d = self.G.det(q)
        return np.concatenate([d.real, d.imag])

    def vjp(self, x, view, rr):
        nn = self.s.n * self.s.n
        r = np.asarray(rr[:nn], float) + 1j * np.asarray(rr[nn:], float)
        f, fp = self.pot(x)
        u, _ = self.total_field(x, view)
        w = self.G.det_adj(r)
        if self.model == "ls":
            cf = np.conj(f)
            z, it, _ = bicgstab(lambda v: v - cf * self.G.dom_adj(v), cf * w, self.tol, self.max_iter)
            self.last_iters.append(it)
            w = w + self.G.dom_adj(z)
        return np.real(np.conj(fp * u) * w)

    def gradient(self, x, view, y):
        return self.vjp(x, view, self.forward(x, view) - y)

    def value(self, x, view, y):
        r = self.forward(x, view) - y
        return 0.5 * float(r @ r)


def ellipsoid_phantom(n, n_shapes, dn_lo, dn_hi, seed):
    """Random ellipsoids (centres U[0.25,0.75]^3, semi-axes U[0.08,0.25], random
    rotation, Delta n ~ U[lo, hi]), later shapes overwrite earlier ones."""
    rng = np.random.default_rng(seed)
    c = (np.arange(n) + 0.5) / n
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    pts = np.stack([x, y, z], axis=-1)
    vol = np.zeros((n, n, n))
    for _ in range(n_shapes):
        ctr = rng.uniform(0.25, 0.75, 3)
        ax = rng.uniform(0.08, 0.25, 3)
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        val = rng.uniform(dn_lo, dn_hi)
        loc = (pts - ctr) @ q
        inside = np.sum((loc / ax) ** 2, axis=-1) <= 1.0
        vol[inside] = val
    return vol.reshape(-1)

"""CPU oracle (fp64 numpy/scipy) for the masked-spectrum view operators.

TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's CPU legs).

Restates /root/reference/pkg/src/tvqn/forward_models.py:
  _dct_flat/_idct_flat :86-91 (scipy.fft.dctn/idctn, norm="ortho" -- the
  arithmetic lives in scipy, pinned version in this image: 1.18.1),
  _smooth_flat :139-150, nonlinear_map/jac_vec/adj_vec :166-183,
  subset_gradient :304-309.  Pinned against the reference's own outputs by
  tests/golden/make_golden.py ("views_*" vectors).
"""

from __future__ import annotations

import numpy as np
import scipy.fft


def _nd(dims, x):
    return np.asarray(x, dtype=float).reshape(tuple(reversed(dims)))


def dct(dims, x, inverse=False):
    a = _nd(dims, x)
    f = scipy.fft.idctn if inverse else scipy.fft.dctn
    return f(a, norm="ortho").reshape(-1)


def smooth(dims, x):
    a = _nd(dims, x).copy()
    nd = len(dims)
    for n in range(nd):  # dims[n] is C-order axis nd-1-n
        if dims[n] == 1:
            continue
        ax = nd - 1 - n
        p = np.moveaxis(a, ax, 0)
        q = np.concatenate([p[:1], p, p[-1:]], axis=0)
        a = np.moveaxis((q[:-2] + q[1:-1] + q[2:]) / 3.0, 0, ax)
    return a.reshape(-1)


class DctView:
    def __init__(self, dims, mask, y, strength):
        self.dims, self.mask, self.y, self.s = tuple(dims), np.asarray(mask, float), np.asarray(y, float), strength

    def forward(self, x):
        x = np.asarray(x, float)
        if self.s == 0.0:
            return self.mask * dct(self.dims, x)
        ax = smooth(self.dims, x)
        return self.mask * dct(self.dims, x + self.s * ax * ax)

    def jvp(self, x, w):
        if self.s == 0.0:
            return self.mask * dct(self.dims, w)
        ax = smooth(self.dims, x)
        return self.mask * dct(self.dims, w + 2.0 * self.s * ax * smooth(self.dims, w))

    def vjp(self, x, z):
        q = dct(self.dims, self.mask * z, inverse=True)
        if self.s == 0.0:
            return q
        ax = smooth(self.dims, x)
        return q + 2.0 * self.s * smooth(self.dims, ax * q)

    def value(self, x):
        r = self.forward(x) - self.y
        return 0.5 * float(r @ r)

    def gradient(self, x):
        return self.vjp(x, self.forward(x) - self.y)


def subset_gradient(views, idx, x):
    g = np.zeros(np.asarray(x).size)
    for i in idx:
        g += views[i].gradient(x)
    return g / len(idx)

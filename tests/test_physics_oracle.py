"""Property tests of the builder-specified Born/LS oracle (no reference exists,
SURVEY F2): these are what pins the physics that the device path must match.
Patterns follow the reference's view tests (tests/test_forward_models.py:77-105)
and ViewProblem.self_check (forward_models.py:66-83).  CPU only."""

import numpy as np
import pytest

from oracle import physics as P


@pytest.fixture(scope="module")
def small():
    s = P.Setup(n=10, n_views=4)
    x = P.ellipsoid_phantom(10, 3, 0.01, 0.05, seed=1)
    return s, x


@pytest.mark.parametrize("model", ["born", "ls"])
def test_adjoint_identity(small, model):
    s, x = small
    m = P.ScatterModel(s, model, tol=1e-12)
    rng = np.random.default_rng(0)
    dx = rng.standard_normal(s.n ** 3)
    rr = rng.standard_normal(2 * s.n ** 2)
    lhs = float(m.jvp(x, 1, dx) @ rr)
    rhs = float(dx @ m.vjp(x, 1, rr))
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))


@pytest.mark.parametrize("model", ["born", "ls"])
def test_gradient_matches_finite_differences(small, model):
    s, x = small
    m = P.ScatterModel(s, model, tol=1e-12)
    y = m.forward(x * 0.8, 2)
    g = m.gradient(x, 2, y)
    rng = np.random.default_rng(1)
    d = rng.standard_normal(s.n ** 3)
    d /= np.linalg.norm(d)
    h = 1e-6
    fd = (m.value(x + h * d, 2, y) - m.value(x - h * d, 2, y)) / (2 * h)
    an = float(g @ d)
    assert abs(fd - an) <= 1e-5 * max(1.0, abs(fd), abs(an))


def test_born_limit(small):
    s, x = small
    ls = P.ScatterModel(s, "ls", tol=1e-13)
    born = P.ScatterModel(s, "born")
    for eps in (1e-3, 1e-4):
        a = ls.forward(eps * x, 0)
        b = born.forward(eps * x, 0)
        rel = np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel < 50 * eps  # O(contrast) relative difference


def test_zero_fidelity_at_truth(small):
    s, x = small
    m = P.ScatterModel(s, "ls", tol=1e-12)
    y = m.forward(x, 3)
    assert m.value(x, 3, y) == 0.0
    assert np.linalg.norm(m.gradient(x, 3, y)) == 0.0


def test_green_convolution_is_aperiodic(small):
    s, _ = small
    G = P.Green(s)
    n = s.n
    v = np.zeros(n ** 3, complex)
    v[0] = 1.0  # voxel (0,0,0)
    out = G.dom(v).reshape(n, n, n)
    # value at (z, y, x) = (0, 0, n-1) equals the kernel at distance (n-1) h
    d = (n - 1) * s.h
    expect = s.h ** 3 * np.exp(1j * s.kb * d) / (4 * np.pi * d)
    assert abs(out[0, 0, n - 1] - expect) < 1e-12 * abs(expect)

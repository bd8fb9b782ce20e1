"""Seeded synthetic inputs for the BASELINE.json configurations.

Seeds follow SURVEY 8d: ``numpy.random.default_rng(1000*c + k)`` for config c,
k = 0 phantom, 1 noise, 2 metric (d, u), 3 prox-volume noise.  No public
dataset is involved; these seeded phantoms stand in for the paper's data.
"""

from __future__ import annotations

import numpy as np


def _rng(config: int, k: int):
    return np.random.default_rng(1000 * config + k)


def box_phantom(n: int, n_boxes: int = 16, rng=None) -> np.ndarray:
    """Piecewise-constant volume of axis-aligned random boxes, later boxes
    overwrite earlier ones; returned flat in Fortran order over (n, n, n)."""
    rng = rng or _rng(2, 0)
    vol = np.zeros((n, n, n))  # C-order (K3, K2, K1) == flat Fortran over dims
    for _ in range(n_boxes):
        side = rng.uniform(n / 16, n / 4, size=3)
        corner = rng.uniform(0, n, size=3)
        val = rng.uniform(0.0, 1.0)
        lo = np.floor(corner).astype(int)
        hi = np.minimum(n, np.floor(corner + side).astype(int) + 1)
        vol[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = val
    return vol.reshape(-1)


def config2_inputs(n: int = 128):
    """Config 2 (weighted-TV prox microbench): v = box phantom + N(0,1) noise,
    W = diag(d) + u u^T with d ~ U[0.5, 2], u ~ N(0,1)/sqrt(N); scalar-tau twin d == 1.25."""
    N = n ** 3
    phantom = box_phantom(n, rng=_rng(2, 0))
    v = phantom + _rng(2, 3).standard_normal(N)
    rm = _rng(2, 2)
    d = rm.uniform(0.5, 2.0, N)
    u = rm.standard_normal(N) / np.sqrt(N)
    return {"n": n, "v": v, "d": d, "u": u, "phantom": phantom, "reg": 0.05, "lo": 0.0, "hi": np.inf,
            "iters": 100, "tau_twin": 1.25}


def ls_phantom(n: int, n_shapes: int, dn_lo: float, dn_hi: float, seed: int) -> np.ndarray:
    """Random ellipsoids for the LS configurations: centres U[0.25,0.75]^3,
    semi-axes U[0.08,0.25], random rotation, dn ~ U[lo, hi], later shapes overwrite."""
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
        inside = np.sum((((pts - ctr) @ q) / ax) ** 2, axis=-1) <= 1.0
        vol[inside] = val
    return vol.reshape(-1)


def cell_phantom(n: int, seed: int, dn_lo: float = 0.005, dn_hi: float = 0.06) -> np.ndarray:
    """Config 5: a cell-like nest of ellipsoids -- membrane shell,
    cytoplasm, nucleus, two nucleoli -- with sorted dn ~ U[lo, hi] (inner levels
    denser), random orientations; later (inner) shapes overwrite outer ones."""
    rng = np.random.default_rng(seed)
    c = (np.arange(n) + 0.5) / n
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    pts = np.stack([x, y, z], axis=-1)
    vol = np.zeros((n, n, n))
    levels = np.sort(rng.uniform(dn_lo, dn_hi, 4))
    ctr = 0.5 + rng.uniform(-0.03, 0.03, 3)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    ax = rng.uniform(0.33, 0.40, 3)

    def fill(centre, axes, rot, val):
        inside = np.sum((((pts - centre) @ rot) / axes) ** 2, axis=-1) <= 1.0
        vol[inside] = val

    fill(ctr, ax, q, levels[1])                 # membrane shell (outer ellipsoid) ...
    fill(ctr, ax - 0.02, q, levels[0])          # ... hollowed by the cytoplasm
    nq, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    nctr = ctr + rng.uniform(-0.06, 0.06, 3)
    nax = ax * rng.uniform(0.35, 0.45, 3)
    fill(nctr, nax, nq, levels[2])              # nucleus
    for _ in range(2):                          # nucleoli
        off = rng.uniform(-0.5, 0.5, 3) * nax
        fill(nctr + off @ nq.T, nax * rng.uniform(0.2, 0.3, 3), nq, levels[3])
    return vol.reshape(-1)


def born_spheres_phantom(n: int, seed: int, n_spheres: int = 3, dn_lo: float = 0.01, dn_hi: float = 0.05):
    """Config 1: 3 random spheres (centres 0.3 + 0.4 U^3, radii linspace(0.32, 0.10, 3)
    (0.8 + 0.4 U) as box fractions -- the reference law, forward_models.py:262-263 --
    with dn ~ U[lo, hi]); later spheres overwrite earlier ones."""
    rng = np.random.default_rng(seed)
    c = (np.arange(n) + 0.5) / n
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    centres = 0.3 + 0.4 * rng.random((n_spheres, 3))
    radii = np.linspace(0.32, 0.10, n_spheres) * (0.8 + 0.4 * rng.random(n_spheres))
    dn = rng.uniform(dn_lo, dn_hi, n_spheres)
    vol = np.zeros((n, n, n))
    for ctr, r, val in zip(centres, radii, dn):
        vol[(x - ctr[0]) ** 2 + (y - ctr[1]) ** 2 + (z - ctr[2]) ** 2 <= r * r] = val
    return vol.reshape(-1)


def complex_noise(y: np.ndarray, snr_db: float, rng) -> np.ndarray:
    """Real-packed [Re; Im] Gaussian noise with 20 log10(||y|| / ||e||) = snr_db."""
    e = rng.standard_normal(y.shape[0])
    return e * (np.linalg.norm(y) / np.linalg.norm(e)) * 10.0 ** (-snr_db / 20.0)

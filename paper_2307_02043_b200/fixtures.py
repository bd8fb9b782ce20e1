"""Host-side input generators: restatements of the reference's mask and phantom laws.

NOT the hot path.  These build the *inputs* of the DCT stand-in views (the
per-view spectrum masks, the nested-sphere phantom) and the SNR reported in
the trace.  They restate the reference's published construction
(``/root/reference/pkg/src/tvqn/forward_models.py``: ``spectrum_masks``
:94-136, ``make_phantom`` :242-282, ``snr_db`` :219-228) because the golden
views are only comparable when the masks are identical bit for bit and the
seeded RNG is consumed in the same order (centres, then radii).  The code is
organised differently (vectorised over views, one angle table), the
arithmetic per element is the same.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .tv_ops import Grid

# widest half-angle of the missing cone (forward_models.py:96)
CONE_MAX_RAD = math.radians(20.0)


def _polar_angle(grid: Grid) -> np.ndarray:
    """Angle between each frequency's normalised position and the last axis (flat order)."""
    ax = [np.arange(k, dtype=float) / max(k - 1, 1) for k in grid.dims]
    coords = np.meshgrid(*ax, indexing="ij")
    transverse = np.sqrt(sum(c * c for c in coords[:-1]))
    return grid.from_nd(np.arctan2(transverse, coords[-1]))


def spectrum_masks(grid: Grid, n_views, mask_fraction):
    """(masks, cone): per-view binary frequency sectors around equispaced polar
    centres, the missing cone removed and the DC term always kept."""
    if n_views < 1:
        raise ValueError("need at least one view")
    if not 0.0 < mask_fraction <= 1.0:
        raise ValueError("mask_fraction must lie in (0, 1]")
    n = grid.size
    dc = np.arange(n) == 0
    if grid.ndim == 1:
        k = np.arange(n)
        return [((k % n_views) == v) | dc for v in range(n_views)], np.zeros(n, dtype=bool)
    ang = _polar_angle(grid)
    phi_cone = CONE_MAX_RAD * (1.0 - mask_fraction)
    cone = (ang < phi_cone) & ~dc
    span = math.pi / 2.0 - phi_cone
    half = span * max(mask_fraction, 1.0 / n_views) / 2.0 + 1e-12
    centres = phi_cone + (np.arange(n_views) + 0.5) * span / n_views
    inside = np.abs(ang[None, :] - centres[:, None]) <= half
    table = (inside & ~cone[None, :]) | dc[None, :]
    return [row for row in table], cone


@dataclass(frozen=True, eq=False)
class Phantom:
    grid: Grid
    values: np.ndarray
    eta_m: float
    eta_max: float
    spheres: tuple


def make_phantom(grid: Grid, kind="spheres", eta_m=1.333, eta_max=1.363, seed=0):
    """Three nested spheres of rising index (or one centred cube) in a medium eta_m."""
    if eta_max < eta_m:
        raise ValueError("eta_max must be >= eta_m")
    rng = np.random.default_rng(seed)
    centres_1d = [(np.arange(k, dtype=float) + 0.5) / k for k in grid.dims]
    pos = np.meshgrid(*centres_1d, indexing="ij")
    vol = np.full(grid.dims, eta_m, dtype=float)
    if kind == "cube":
        inside = np.logical_and.reduce([(p > 0.3) & (p < 0.7) for p in pos])
        vol[inside] = eta_max
        shapes = (((0.5,) * grid.ndim, 0.2, eta_max),)
    elif kind == "spheres":
        count = 3
        level = eta_m + (eta_max - eta_m) * np.linspace(1.0 / count, 1.0, count)
        ctr = 0.3 + 0.4 * rng.random((count, grid.ndim))          # RNG draw 1
        rad = np.linspace(0.32, 0.10, count) * (0.8 + 0.4 * rng.random(count))  # RNG draw 2
        shapes = []
        for i in range(count):  # later spheres overwrite earlier ones
            dist2 = sum((pos[a] - ctr[i, a]) ** 2 for a in range(grid.ndim))
            vol[dist2 <= rad[i] * rad[i]] = level[i]
            shapes.append((tuple(ctr[i]), float(rad[i]), float(level[i])))
        shapes = tuple(shapes)
    else:
        raise ValueError(f"unknown phantom kind: {kind!r}")
    return Phantom(grid=grid, values=grid.from_nd(vol), eta_m=eta_m, eta_max=eta_max, spheres=shapes)


def _host(a) -> np.ndarray:
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy().astype(float)
    return np.asarray(a, dtype=float)


def snr_db(x, x_ref):
    """20 log10(||x_ref|| / ||x - x_ref||) (inf for an exact match)."""
    x, x_ref = _host(x), _host(x_ref)
    if x.shape != x_ref.shape:
        raise ValueError("shapes must match")
    err = float(np.linalg.norm(x - x_ref))
    return math.inf if err == 0.0 else 20.0 * math.log10(float(np.linalg.norm(x_ref)) / err)


__all__ = ["CONE_MAX_RAD", "spectrum_masks", "Phantom", "make_phantom", "snr_db"]

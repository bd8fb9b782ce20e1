"""End-to-end BQNPM runs on the device loop (wall clock, host control included).

(a) the reference's own stand-in: DCT views, 32^3, L=16, K_s=4, 20 outer
    iterations, lambda 1e-3, box [0, 0.1], fp64 -- the run SURVEY 6 timed on the
    reference (4.93 s on one CPU core, 80% in the prox);
(b) BASELINE config 1: first-Born views, 32^3, c128, L=16, K_s=4, 20 outer
    iterations, lambda 1e-3, box [0, 0.1].
Each run includes the Lipschitz startup and the default initializer; view
construction and measurement synthesis are excluded.

    python bench/loop_bench.py [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_02043_b200 import physics as PH  # noqa: E402
from paper_2307_02043_b200 import solvers as S  # noqa: E402
from paper_2307_02043_b200.configs import born_spheres_phantom  # noqa: E402
from paper_2307_02043_b200.forward_models import make_linear_views, make_phantom  # noqa: E402
from paper_2307_02043_b200.tv_ops import Grid  # noqa: E402
from paper_2307_02043_b200.wpm import BoxSet  # noqa: E402


def timed_run(views, grid, cfg, xgt, reps):
    S.bqnpm_run(views, grid, cfg, ground_truth=xgt)  # warm-up (plans, workspaces)
    ts, tr = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, tr = S.bqnpm_run(views, grid, cfg, ground_truth=xgt)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    inner = tr.column("inner_iters")[1:]
    return {"s_total": float(np.median(ts)), "ms_per_outer": 1e3 * float(np.median(ts)) / cfg.max_outer,
            "mean_fgp_iters": float(np.mean(inner)), "final_cost": float(tr.final_cost),
            "final_snr_db": float(tr.rows[-1].snr_db)}


def measure(reps=3):
    out = {"note": "wall clock of bqnpm_run incl. Lipschitz startup + initializer, view construction excluded"}
    n = 32
    grid = Grid((n, n, n))
    xgt = make_phantom(grid, seed=0).values - 1.333  # the reference's nested spheres, as dn in [0, 0.03]
    views = make_linear_views(grid, 16, seed=1001, x_gt=xgt, noise_snr_db=30.0)
    cfg = S.SolverConfig(subsets=4, tv_weight=1e-3, max_outer=20, box=BoxSet(0.0, 0.1), seed=0)
    out["dct_32_L16_bqnpm20"] = timed_run(views, grid, cfg, xgt, reps)
    out["dct_32_L16_bqnpm20"]["reference_cpu_s"] = 4.93  # SURVEY 6, measured on the reference in the survey container
    xgt1 = born_spheres_phantom(n, seed=1000)
    views1, _ = PH.make_scatter_views(n, 16, model="born", x_gt=xgt1, noise_snr_db=30.0, seed=1001,
                                      dtype=torch.complex128, theta_deg=35.0, batch=8)
    out["config1_born_32_L16_bqnpm20"] = timed_run(views1, grid, cfg, xgt1, reps)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    print(json.dumps(measure(args.reps)))


if __name__ == "__main__":
    main()

"""Full-size BQNPM reconstructions of BASELINE configs 3, 4 and 5 on ONE GPU (wall clock).

  config 3: LS, n = 64 (128^3 padded), c64, L = 32, batch 8, BiCGSTAB tol 1e-6, 5 ellipsoids dn in [0.02, 0.08],
            30 dB noise, 30 outer iterations
  config 4: LS, n = 128 (256^3 padded), c64, L = 64 on a 40-degree cone, batch 16, 12 ellipsoids dn in [0.01, 0.1],
            25 dB noise (outer iterations: --outer4, default 20)
  config 5: LS, n = 256 (512^3 padded), c64, L = 120, subsets of 30 views, cell phantom dn in [0.005, 0.06],
            25 dB noise, 20 outer iterations (the prox runs the fused single-GPU kernel here; the z-slab path
            is for N > 1 ranks)

Synthetic seeded phantoms stand in for the paper's data (configs.py).  lambda = 1e-3 and box [0, 0.1] as in
config 1; the initial guess is the scaled adjoint step (DESIGN D-8).  Reported per config: measurement synthesis,
startup (initial guess + Lipschitz constants) and outer-iteration times, the cost and SNR trace ends.

    python bench/recon_bench.py --configs 3 4 [5]
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
from paper_2307_02043_b200.configs import cell_phantom, ls_phantom  # noqa: E402
from paper_2307_02043_b200.forward_models import snr_db  # noqa: E402
from paper_2307_02043_b200.tv_ops import Grid  # noqa: E402
from paper_2307_02043_b200.wpm import BoxSet  # noqa: E402

CONFIGS = {
    3: dict(n=64, views=32, batch=8, theta=35.0, snr=30.0, outer=30, trace_every=1, phantom=lambda n: ls_phantom(n, 5, 0.02, 0.08, seed=3000)),
    4: dict(n=128, views=64, batch=16, theta=40.0, snr=25.0, outer=20, trace_every=5, phantom=lambda n: ls_phantom(n, 12, 0.01, 0.1, seed=4000)),
    5: dict(n=256, views=120, batch=30, theta=40.0, snr=25.0, outer=20, trace_every=10, phantom=lambda n: cell_phantom(n, seed=5000)),
}


def sync():
    torch.cuda.synchronize()
    return time.perf_counter()


def run(k, outer=None, power_iters=4, dn_hi=None):
    c = CONFIGS[k]
    n = c["n"]
    outer = outer or c["outer"]
    xgt = c["phantom"](n)
    if dn_hi is not None:  # same shapes at a lower peak contrast (config 4 is strongly scattering as specified)
        xgt = xgt * (dn_hi / float(xgt.max()))
    t0 = sync()
    views, vs = PH.make_scatter_views(n, c["views"], model="ls", x_gt=xgt, noise_snr_db=c["snr"], seed=1000 * k + 1,
                                      dtype=torch.complex64, theta_deg=c["theta"], batch=c["batch"], tol=1e-6,
                                      max_iter=500)
    t1 = sync()
    grid = Grid((n, n, n))
    box = BoxSet(0.0, 0.1)
    nsub = c["views"] // c["batch"]
    x0 = S.scaled_adjoint_initializer(views, grid, box)
    parts = S.partition_views(len(views), nsub)
    al = S.estimate_subset_lipschitz(views, parts, x0, power_iters, 1.05, 0)
    t2 = sync()
    # the full cost over all L views is a reporting step (L forward solves): every trace_every iterations
    cfg = S.SolverConfig(subsets=nsub, tv_weight=1e-3, max_outer=outer, box=box, seed=0, alphas=al,
                         trace_every=c["trace_every"])
    x, tr = S.bqnpm_run(views, grid, cfg, x0=x0, ground_truth=xgt)
    t3 = sync()
    xh = x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)
    cost = tr.column("cost")
    snr = tr.column("snr_db")
    return {"config": k, "dn_max": float(xgt.max()), "n": n, "views": c["views"], "subset": c["batch"], "outer_iterations": outer,
            "synthesis_s": t1 - t0, "startup_s": t2 - t1, "iterations_s": t3 - t2,
            "s_per_outer": (t3 - t2) / outer, "lipschitz_power_iters": power_iters, "trace_every": c["trace_every"],
            "cost_first": float(cost[0]), "cost_last": float(cost[-1]),
            "snr_db_first": float(snr[0]), "snr_db_last": float(snr[-1]),
            "snr_db_ri_map_last": float(snr_db(1.333 + xh, 1.333 + xgt)),
            "mean_fgp_iters": float(np.mean(tr.column("inner_iters")[1:])),
            "mean_bicgstab_forward": float(np.mean(vs.iters_forward)) if vs.iters_forward else None,
            "mean_bicgstab_adjoint": float(np.mean(vs.iters_adjoint)) if vs.iters_adjoint else None,
            "gpu_mem_peak_gb": torch.cuda.max_memory_allocated() / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
    ap.add_argument("--outer", type=int, default=0, help="override the outer iteration count")
    ap.add_argument("--dn-hi", type=float, default=0.0, help="rescale the phantom to this peak contrast")
    args = ap.parse_args()
    for k in args.configs:
        torch.cuda.reset_peak_memory_stats()
        print(json.dumps(run(k, args.outer or None, dn_hi=args.dn_hi or None)), flush=True)


if __name__ == "__main__":
    main()

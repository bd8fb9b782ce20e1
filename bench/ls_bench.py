"""LS forward+adjoint throughput (BASELINE configs 3/4): one subset gradient of
`batch` views = batched forward BiCGSTAB + detector + adjoint BiCGSTAB + grad.

    python bench/ls_bench.py --n 128 --views 64 --batch 16 --theta 40 --steps 2
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
from paper_2307_02043_b200.configs import ls_phantom as ellipsoid_phantom  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--theta", type=float, default=40.0)
    ap.add_argument("--shapes", type=int, default=12)
    ap.add_argument("--dn", type=float, nargs=2, default=[0.01, 0.1])
    ap.add_argument("--snr", type=float, default=25.0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--max-iter", type=int, default=500)
    args = ap.parse_args()
    n = args.n
    xgt = ellipsoid_phantom(n, args.shapes, args.dn[0], args.dn[1], seed=4000)
    t0 = time.time()
    views, vs = PH.make_scatter_views(n, args.views, model="ls", x_gt=xgt, noise_snr_db=args.snr, seed=4001,
                                      theta_deg=args.theta, batch=args.batch, max_iter=args.max_iter)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    # evaluate at a mid-reconstruction state (x = 0 makes A the identity: 1 iteration)
    x = torch.tensor(0.5 * xgt, dtype=torch.float32, device="cuda")
    idx = list(range(0, args.views, args.views // args.batch))[: args.batch]
    vs.subset_gradient(idx, x)  # warm-up (plans)
    times = []
    kf, ka = [], []
    for _ in range(args.steps):
        vs.iters_forward.clear()
        vs.iters_adjoint.clear()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        g = vs.subset_gradient(idx, x)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
        kf.append(np.mean(vs.iters_forward))
        ka.append(np.mean(vs.iters_adjoint))
    ms = float(np.median(times))
    Kf, Ka = float(np.mean(kf)), float(np.mean(ka))
    pruned = (2 * n) in (16, 32, 64, 128, 256, 512) and os.environ.get("BQ_LS_CUFFT", "0") != "1"
    bytes_vv = (2.0 * (220.0 if pruned else 412.0) + 128.0) * (Kf + Ka) + 92.0  # SURVEY 8d, pruned matvec bytes (bench.py)
    vv = len(idx) * n ** 3
    out = {"metric": "LS forward+adjoint views*voxels/s", "n": n, "views_in_subset": len(idx), "ms": ms,
           "value": vv / (ms * 1e-3), "K_f": Kf, "K_a": Ka, "bytes_per_view_voxel": bytes_vv,
           "achieved_GBps": vv * bytes_vv / (ms * 1e-3) / 1e9, "setup_s": setup_s,
           "grad_norm": float(torch.linalg.vector_norm(g).item())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

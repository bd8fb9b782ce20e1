#!/usr/bin/env python
"""Benchmark of the BQNPM hot path on B200 (driver contract: ONE JSON line on rank 0).

Headline workload = BASELINE.json configs[1] (config 2): the weighted-TV prox
microbench, 128^3 fp32, W = diag(d) + u u^T, isotropic TV reg 0.05, box
[0, inf), exactly 100 FGP iterations (eps = 1e-300), P0 = 0, beta0 = 0.
A "step" is one full prox solve (one persistent-kernel launch).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 128]

--impl reference times the CPU restatement of the reference algorithm
(oracle/prox.py, the reference package itself cannot travel to the GPU box)
on a bounded sample of the same workload; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "wTV-prox voxel-iters/s"
UNIT = "voxel*iter/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def bytes_per_voxel_iter(word: int, rank: int, per_voxel_d: bool) -> int:
    """B_wtv = s * (13 + r + delta_d): read P_bar, P, write P, P_bar
    (3 each), read v, U (r), d (per-voxel)."""
    return word * (13 + rank + (1 if per_voxel_d else 0))


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML,
    every 5 ms; nvidia-smi CLI fallback)."""

    REASONS = {  # nvmlClocksEventReasons bits
        "sw_power_cap": 0x4,
        "hw_slowdown": 0x8,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.sm = []
        self.max_sm = None
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for name, bit in self.REASONS.items():
            if bits & bit:
                self.reasons.add(name)

    def _sample_cli(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip().split(",")
        self.sm.append(float(out[0]))
        self.max_sm = float(out[1])
        bits = int(out[2], 16)
        for name, bit in self.REASONS.items():
            if bits & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_cli()
            except Exception:
                pass
            self._stop.wait(self.period if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: CPU restatement on the host cores
# ---------------------------------------------------------------------------
def cpu_prox_sample(inp, iters: int):
    from oracle import prox as O

    n = inp["n"]
    w = O.Metric(U=inp["u"][:, None], d=inp["d"])
    t0 = time.perf_counter()
    O.fgp_prox((n, n, n), inp["v"], w, reg=inp["reg"], eps=1e-300, max_iter=iters)
    dt = time.perf_counter() - t0
    return n ** 3 * iters / dt, dt


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2307_02043_b200.configs import config2_inputs

    inp = config2_inputs(args.n)
    vals = []
    sample_iters = args.cpu_iters
    for _ in range(args.warmup):
        cpu_prox_sample(inp, 1)
    t_all = time.perf_counter()
    for _ in range(args.steps):
        v, _ = cpu_prox_sample(inp, sample_iters)
        vals.append(v)
    wall = time.perf_counter() - t_all
    value = float(np.median(vals))
    sample = f"config-2 prox {args.n}^3 f64 diag(d)+uu^T, {sample_iters} FGP iterations per step (numpy port)"
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-2 box phantom + N(0,1) noise)",
        # the same workload as the device arm (a voxel*iter of one 100-iteration solve);
        # each step times a bounded sample of its FGP iterations
        "config": {"workload": f"config2 wTV prox {args.n}^3 W=diag(d)+uu^T iso TV reg 0.05 box [0,inf), "
                               f"100 FGP iterations per step",
                   "sample_iters_per_step": sample_iters, "parallelism": "host cores x1 (numpy port)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# e2e: host (pinned) buffers through the public API, copies inside the timed region
# ---------------------------------------------------------------------------
def _e2e_problem(grid, inp, v, d, u):
    from paper_2307_02043_b200 import dual_tv_solver as D
    from paper_2307_02043_b200.wpm import BoxSet, DiagPlusLowRank

    w = DiagPlusLowRank(1.0, u[:, None], d=d)  # validates d > 0 and W PD (host syncs)
    return D.DualTvProblem(grid=grid, v=v, w=w, reg=inp["reg"], box=BoxSet(0.0, np.inf))


def e2e_serial_ms(args, dev, grid, inp, wsp, v_h, d_h, u_h, iters):
    """One step at a time: H2D, build, solve, D2H, synchronize."""
    import torch
    from paper_2307_02043_b200 import dual_tv_solver as D

    out_h = torch.empty(v_h.numel(), dtype=wsp.dtype).pin_memory()
    ms = []
    for i in range(args.steps + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        pp = _e2e_problem(grid, inp, v_h.to(dev, non_blocking=True), d_h.to(dev, non_blocking=True),
                          u_h.to(dev, non_blocking=True))
        D.solve_async(pp, wsp, eps=1e-300, max_iter=iters)
        out_h.copy_(wsp.x, non_blocking=True)
        torch.cuda.synchronize(dev)
        if i > 0:
            ms.append(1e3 * (time.perf_counter() - t0))
    return float(np.mean(ms))


def e2e_pipelined_ms(args, dev, grid, inp, wsp, v_h, d_h, u_h, iters, slots=3):
    """Three input slots and workspaces.  Right after solve i is queued, step
    i+1's inputs stream in on a high-priority side stream and its problem is
    built and validated there (DiagPlusLowRank / DualTvProblem through the
    public API, validation syncs included): the copies overlap solve i-1, the
    validation kernels take the SMs between solve i-1 and solve i, so solve i+1
    is queued before solve i ends.  x_i streams out on a D2H stream under solve
    i+1 and the host reads every step's x."""
    import torch
    from paper_2307_02043_b200 import dual_tv_solver as D

    main = torch.cuda.current_stream(dev)
    s_in = torch.cuda.Stream(dev, priority=-1)
    s_out = torch.cuda.Stream(dev)
    N = v_h.numel()
    bufs = [[torch.empty_like(t, device=dev) for t in (v_h, d_h, u_h)] for _ in range(slots)]
    wsps = [wsp] + [D.ProxWorkspace(grid, wsp.dtype, dev) for _ in range(slots - 1)]
    outs = [torch.empty(N, dtype=wsp.dtype).pin_memory() for _ in range(slots)]
    probs = [None] * slots  # held until the slot is reused (their tensors live on s_in)
    ev_in = [torch.cuda.Event() for _ in range(slots)]
    ev_done = [torch.cuda.Event() for _ in range(slots)]
    ev_out = [torch.cuda.Event() for _ in range(slots)]
    used = [False] * slots
    checks = []

    def build(i):
        s = i % slots
        with torch.cuda.stream(s_in):
            if used[s]:
                s_in.wait_event(ev_done[s])  # the solve that read this slot (step i-slots) is done
            for dst, src in zip(bufs[s], (v_h, d_h, u_h)):
                dst.copy_(src, non_blocking=True)
            probs[s] = _e2e_problem(grid, inp, *bufs[s])  # its syncs wait on s_in only
            ev_in[s].record(s_in)

    def run(total):
        build(0)
        for i in range(total):
            s = i % slots
            main.wait_event(ev_in[s])
            if used[s]:
                ev_out[s].synchronize()  # host has x_{i-slots}; slot s's workspace and output are free
                checks.append(float(outs[s][N // 2]))
            D.solve_async(probs[s], wsps[s], eps=1e-300, max_iter=iters)
            ev_done[s].record(main)
            used[s] = True
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[s])
                outs[s].copy_(wsps[s].x, non_blocking=True)
                ev_out[s].record(s_out)
            if i + 1 < total:
                build(i + 1)
        for s in range(slots):
            if used[s]:
                ev_out[s].synchronize()
                checks.append(float(outs[s][N // 2]))

    run(max(args.warmup, 3))
    torch.cuda.synchronize(dev)
    used[:] = [False] * slots
    t0 = time.perf_counter()
    run(args.steps)
    torch.cuda.synchronize(dev)
    ms = 1e3 * (time.perf_counter() - t0) / args.steps
    ref = wsp.x.float().cpu()
    if not all(c == checks[0] for c in checks) or checks[0] != float(ref[N // 2]):
        raise RuntimeError("pipelined e2e: a step's x differs from the resident solve")
    return ms


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    # BQ_BENCH_SHARE_GPU=1: functional check of the N>1 code path on one GPU
    # (gloo, all ranks on device 0) -- never a measurement
    share = os.environ.get("BQ_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_2307_02043_b200 as bq
    from paper_2307_02043_b200 import dual_tv_solver as D
    from paper_2307_02043_b200.configs import config2_inputs
    from paper_2307_02043_b200.wpm import BoxSet, DiagPlusLowRank

    n = args.n
    N = n ** 3
    dtype = torch.float32
    inp = config2_inputs(n)
    grid = bq.Grid((n, n, n))
    v_h = torch.from_numpy(inp["v"].astype(np.float32)).pin_memory()
    d_h = torch.from_numpy(inp["d"].astype(np.float32)).pin_memory()
    u_h = torch.from_numpy(inp["u"].astype(np.float32)).pin_memory()
    v = v_h.to(dev)
    d = d_h.to(dev)
    u = u_h.to(dev)
    w = DiagPlusLowRank(1.0, u[:, None], d=d)
    prob = D.DualTvProblem(grid=grid, v=v, w=w, reg=inp["reg"], box=BoxSet(0.0, np.inf))
    wsp = D.ProxWorkspace(grid, dtype, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2
    iters = inp["iters"]

    def step():
        D.solve_async(prob, wsp, eps=1e-300, max_iter=iters)

    for _ in range(max(args.warmup, 3)):
        step()
    rep = D.read_report(wsp)
    assert rep.iterations == iters, rep.iterations

    stream = torch.cuda.current_stream(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with sampler:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 between timed steps (not inside the event pair)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t_wall
    if ws > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    last = D.read_report(wsp)
    names = ["setup", "div", "newton_full", "fused", "final", "newton_local"]
    phases = {nm: {"ms": last.phase_ns[i] / 1e6, "work_ms": last.phase_work_ns[i] / 1e6,
                   "visits": int(last.phase_count[i])} for i, nm in enumerate(names)}
    ms = float(np.mean(step_ms))
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ws * N * iters / (ms * 1e-3)

    # ---- e2e: host buffers through the public API, copies inside the timed region
    e2e_serial = e2e_serial_ms(args, dev, grid, inp, wsp, v_h, d_h, u_h, iters)
    e2e = e2e_pipelined_ms(args, dev, grid, inp, wsp, v_h, d_h, u_h, iters)
    if ws > 1:
        t = torch.tensor([e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    ls = None
    if not args.no_ls:
        ls = ls_measure(args, dev, ws)  # collective at N > 1
    more = None
    if rank == 0 and not args.no_more:
        more = prox_variants(dev, flush)
    loop = None
    if rank == 0 and not args.no_loop:
        sys.path.insert(0, str(ROOT / "bench"))
        import loop_bench

        loop = loop_bench.measure(reps=2)

    if rank == 0:
        peak, peak_kind = hbm_peak()
        bpv = bytes_per_voxel_iter(4, 1, True)
        achieved = bpv * N * iters / (ms * 1e-3) / 1e9
        traffic = None
        summ = ROOT / "profiles" / "ncu_summary.json"
        if summ.exists():
            try:
                traffic = json.loads(summ.read_text()).get("wtv_prox_kernel", {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        cpu = None
        if ws == 1 and not args.no_cpu:
            inp64 = inp
            cv, cdt = cpu_prox_sample(inp64, args.cpu_iters)
            cpu = {"value": cv, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"config-2 prox {n}^3 f64 diag(d)+uu^T, {args.cpu_iters} FGP iterations "
                             f"(numpy port, {cdt:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded config-2 box phantom + N(0,1) noise)",
            "config": {"workload": f"config2 wTV prox {n}^3 W=diag(d)+uu^T iso TV reg 0.05 box [0,inf), "
                                   f"{iters} FGP iterations per step",
                       "l2": "flushed (256 MB write) between timed steps", "parallelism": f"replicas x{ws}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind, "algorithmic_bytes_per_voxel_iter": bpv},
            "cpu_baseline": cpu,
            "e2e": {"value": ws * N * iters / (e2e * 1e-3), "unit": UNIT, "ms_per_step": e2e,
                    "h2d_bytes_per_step": 3 * N * 4, "d2h_bytes_per_step": N * 4,
                    "schedule": "pipelined, 3 slots: step i+1's H2D (v, d, u) and its DiagPlusLowRank / "
                                "DualTvProblem build (validation syncs included) run on a high-priority side "
                                "stream under solve i-1, x_i's D2H on a copy stream under solve i+1; the host "
                                "reads every x; wall clock over all steps",
                    "serial_ms_per_step": e2e_serial},
            "gpu_launches": args.steps,
            "ls": ls,
            "prox_more": more,
            "bqnpm_loop": loop,
            "clocks": sampler.summary(),
            "wall_s_timed_region": wall,
            "prox_phases_last_step": phases,
            "newton_steps_last_step": int(last.newton_iterations),
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def prox_variants(dev, flush):
    """Secondary prox shapes (reported beside the headline, not the headline):
    the config-2 law at 256^3 (config 5's grid, x-split rows) and the BQNPM
    metric W = tau I + U U^T with rank 4 (K_s = 4) at 128^3 and 256^3.  Each:
    3 warm-up solves, 5 timed solves of 100 FGP iterations, L2 flushed between."""
    import torch

    import paper_2307_02043_b200 as bq
    from paper_2307_02043_b200 import dual_tv_solver as D
    from paper_2307_02043_b200.configs import config2_inputs
    from paper_2307_02043_b200.wpm import BoxSet, DiagPlusLowRank

    peak, _ = hbm_peak()
    out = []
    cache = {}
    for n, r, diag in [(256, 1, True), (128, 4, False), (256, 4, False)]:
        if n not in cache:
            cache[n] = config2_inputs(n)
        inp = cache[n]
        N = n ** 3
        v = torch.from_numpy(inp["v"].astype(np.float32)).to(dev)
        if diag:
            w = DiagPlusLowRank(1.0, torch.from_numpy(inp["u"].astype(np.float32)).to(dev)[:, None],
                                d=torch.from_numpy(inp["d"].astype(np.float32)).to(dev))
        else:
            g = torch.Generator(device="cpu").manual_seed(2000 + r)
            U = (torch.randn(N, r, generator=g) / np.sqrt(N)).to(dev)
            w = DiagPlusLowRank(inp["tau_twin"], U)
        prob = D.DualTvProblem(grid=bq.Grid((n, n, n)), v=v, w=w, reg=inp["reg"], box=BoxSet(0.0, np.inf))
        wsp = D.ProxWorkspace(prob.grid, torch.float32, dev)
        for _ in range(3):
            D.solve_async(prob, wsp, eps=1e-300, max_iter=100)
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            D.solve_async(prob, wsp, eps=1e-300, max_iter=100)
            e.record()
            torch.cuda.synchronize(dev)
            ts.append(s.elapsed_time(e))
        ms = float(np.median(ts))
        bpv = bytes_per_voxel_iter(4, r, diag)
        achieved = bpv * N * 100 / (ms * 1e-3) / 1e9
        out.append({"workload": f"{n}^3 fp32 rank {r} " + ("diag(d)+uu^T (config-2 law)" if diag else
                                                           "tau I + U U^T (BQNPM metric)") + ", 100 FGP iterations",
                    "ms_per_solve": ms, "value": N * 100 / (ms * 1e-3), "unit": UNIT,
                    "roofline": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                                 "algorithmic_bytes_per_voxel_iter": bpv}})
        del prob, wsp, w, v
    return out


def ls_measure(args, dev, ws=1):
    """Secondary metric (BASELINE 'views*voxels/s of LS forward+adjoint'): one
    subset gradient of config 4 (n=128 padded to 256^3, c64, 16 of 64 views on a
    40 deg cone, 12 ellipsoids dn~U[0.01,0.1], 25 dB) at x = x_gt / 2."""
    import torch

    from paper_2307_02043_b200 import physics as PH
    from paper_2307_02043_b200.configs import ls_phantom

    n = args.ls_n
    xgt = ls_phantom(n, 12, 0.01, 0.1, seed=4000)
    views, vs = PH.make_scatter_views(n, 64, model="ls", x_gt=xgt, noise_snr_db=25.0, seed=4001, theta_deg=40.0,
                                      batch=16, max_iter=500, device=dev)
    x = torch.tensor(0.5 * xgt, dtype=torch.float32, device=dev)
    idx = list(range(0, 64, 4))
    if ws > 1:
        # view-sharded: each rank takes a contiguous chunk of the subset,
        # one NCCL all-reduce of the gradient; the time is the max over ranks
        import torch.distributed as dist

        from paper_2307_02043_b200 import dist as DI

        def grad():
            return DI.subset_gradient(vs, idx, x)
    else:
        def grad():
            return vs.subset_gradient(idx, x)
    grad()  # plans, warm-up
    times, kf, ka = [], [], []
    for _ in range(max(1, args.ls_steps)):
        vs.iters_forward.clear()
        vs.iters_adjoint.clear()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        s.record()
        grad()
        e.record()
        torch.cuda.synchronize(dev)
        t_ms = s.elapsed_time(e)
        if ws > 1:
            tt = torch.tensor([t_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        times.append(t_ms)
        kf.append(float(np.mean(vs.iters_forward)) if vs.iters_forward else 0.0)
        ka.append(float(np.mean(vs.iters_adjoint)) if vs.iters_adjoint else 0.0)
    ms = float(np.median(times))
    Kf, Ka = float(np.mean(kf)), float(np.mean(ka))
    # bytes per view*voxel = (2 B_mv + 128) (K_f + K_a) + 92, with B_mv the
    # bytes of one padded Green matvec.  SURVEY's 412 N assumes unpruned 3-D
    # transforms; the pruned line passes (csrc/ls_fft.cu) move
    # R 116 N + W 104 N = 220 N, so the count is lowered as 8d requires.
    pruned = (2 * n) in (16, 32, 64, 128, 256, 512) and os.environ.get("BQ_LS_CUFFT", "0") != "1"
    b_mv = 220.0 if pruned else 412.0
    bpv = (2.0 * b_mv + 128.0) * (Kf + Ka) + 92.0
    vv = len(idx) * n ** 3
    peak, _ = hbm_peak()
    peak *= ws  # whole-job bytes over ws GPUs
    achieved = vv * bpv / (ms * 1e-3) / 1e9
    return {"metric": "LS forward+adjoint views*voxels/s", "value": vv / (ms * 1e-3), "unit": "view*voxel/s",
            "ms_per_subset_gradient": ms, "views": len(idx), "n": n, "padded": 2 * n, "dtype": "c64",
            "n_gpus": ws, "scaling": "strong", "parallelism": f"view-sharded x{ws}, one all-reduce",
            "K_f": Kf, "K_a": Ka,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "algorithmic_bytes_per_view_voxel": bpv, "bytes_per_matvec_per_voxel": b_mv,
                         "green_path": "pruned line passes" if pruned else "padded cuFFT"},
            "data": "synthetic (seeded ellipsoid phantom, 25 dB noise), x = x_gt/2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--cpu-iters", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ls", action="store_true")
    ap.add_argument("--no-more", action="store_true", help="skip the secondary prox shapes (256^3, rank 4)")
    ap.add_argument("--no-loop", action="store_true", help="skip the end-to-end BQNPM loop runs (bench/loop_bench.py)")
    ap.add_argument("--ls-n", type=int, default=128)
    ap.add_argument("--ls-steps", type=int, default=2)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

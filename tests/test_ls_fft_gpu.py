"""Pruned padded-Green convolution passes (csrc/ls_fft.cu) against the CPU oracle's
Green operators (oracle/physics.py Green.dom / dom_adj / det / det_adj), every op of
bq_ls_conv, both precisions, every instantiated padded size up to 256; the 512 size
is checked against the cuFFT path of the same library (BQ_LS_CUFFT=1, subprocess)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import physics as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(n, B, seed):
    rng = np.random.default_rng(seed)
    N = n ** 3
    f = rng.uniform(0.0, 3.0, N)
    v = rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))
    r = rng.standard_normal((B, n * n)) + 1j * rng.standard_normal((B, n * n))
    ad = rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))
    return f, v, r, ad


def _oracle(n, op, f, v, r, ad, alpha, beta):
    G = P.Green(P.Setup(n=n))
    out = []
    for b in range(v.shape[0]):
        if op == 0:
            out.append(alpha * v[b] + beta * G.dom(f * v[b]) + ad[b])
        elif op == 1:
            out.append(alpha * v[b] + beta * f * G.dom_adj(v[b]) + ad[b])
        elif op == 2:
            out.append(G.det(f * v[b]))
        else:
            out.append(G.det_adj(r[b]) + ad[b])
    return np.array(out)


def _device(n, op, f, v, r, ad, alpha, beta, cdtype):
    from paper_2307_02043_b200 import physics as PH

    vs = PH.ScatterViewSet(n, 2, model="ls", dtype=cdtype, batch=v.shape[0])
    rt = vs.rdtype
    ft = torch.tensor(f, dtype=rt, device="cuda")
    vin = torch.tensor(r if op == 3 else v, dtype=cdtype, device="cuda")
    adt = None if op == 2 else torch.tensor(ad, dtype=cdtype, device="cuda")
    out = vs.conv(op, ft, vin, alpha=alpha, beta=beta, addend=adt)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("n", [8, 16, 32, 64])
@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_pruned_conv_c128_matches_oracle(n, op):
    f, v, r, ad = _inputs(n, 3, seed=100 + n + op)
    got = _device(n, op, f, v, r, ad, 0.7, -1.3, torch.complex128)
    ref = _oracle(n, op, f, v, r, ad, 0.7, -1.3)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err < 1e-12, (n, op, err)


@pytest.mark.parametrize("n", [16, 64, 128])
@pytest.mark.parametrize("op", [0, 1, 2, 3])
def test_pruned_conv_c64_matches_oracle(n, op):
    f, v, r, ad = _inputs(n, 2 if n < 128 else 1, seed=200 + n + op)
    got = _device(n, op, f, v, r, ad, 1.0, -1.0, torch.complex64)
    ref = _oracle(n, op, f, v, r, ad, 1.0, -1.0)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err < 2e-6, (n, op, err)


def test_non_power_of_two_sizes_use_cufft_path_and_agree():
    n = 12  # padded 24: no pruned instantiation -> cuFFT path
    f, v, r, ad = _inputs(n, 2, seed=5)
    for op in range(4):
        got = _device(n, op, f, v, r, ad, 1.0, -1.0, torch.complex128)
        ref = _oracle(n, op, f, v, r, ad, 1.0, -1.0)
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


_SUB = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2307_02043_b200 import physics as PH
n, op = {n}, {op}
rng = np.random.default_rng(9)
vs = PH.ScatterViewSet(n, 2, model="ls", dtype=torch.complex64, batch=1)
f = torch.tensor(rng.uniform(0, 3, n ** 3), dtype=torch.float32, device="cuda")
L = n * n if op == 3 else n ** 3
v = torch.complex(torch.tensor(rng.standard_normal((1, L)), dtype=torch.float32),
                  torch.tensor(rng.standard_normal((1, L)), dtype=torch.float32)).cuda()
out = vs.conv(op, f, v, alpha=1.0, beta=-1.0)
np.save({path!r}, out.cpu().numpy())
"""


@pytest.mark.parametrize("op", [0, 3])
def test_pruned_conv_512_matches_cufft_path(tmp_path, op):
    n = 256
    res = {}
    for mode in ("pruned", "cufft"):
        path = str(tmp_path / f"{mode}.npy")
        env = dict(os.environ)
        env["BQ_LS_CUFFT"] = "1" if mode == "cufft" else "0"
        code = _SUB.format(root=ROOT, n=n, op=op, path=path)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
        res[mode] = np.load(path)
    err = np.linalg.norm(res["pruned"] - res["cufft"]) / np.linalg.norm(res["cufft"])
    assert err < 2e-6, err


@pytest.mark.parametrize("adjoint", [False, True])
@pytest.mark.parametrize("n", [12, 16])
def test_device_bicgstab_matches_oracle_iterates(adjoint, n):
    """bq_ls_bicgstab (device recurrences, fused dots, skipped converged views) against
    oracle/physics.py bicgstab view by view: same solution and iteration counts, for
    A (forward) and A^H (adjoint), on the pruned (n=16) and cuFFT (n=12) paths."""
    from paper_2307_02043_b200 import physics as PH

    B = 3
    s = P.Setup(n=n)
    G = P.Green(s)
    rng = np.random.default_rng(40 + n + int(adjoint))
    f = rng.uniform(0.0, 60.0, n ** 3) * (rng.uniform(0, 1, n ** 3) < 0.4)
    bs = rng.standard_normal((B, n ** 3)) + 1j * rng.standard_normal((B, n ** 3))
    bs[1] = np.exp(1j * np.arange(n ** 3) * 0.01)  # a smooth right-hand side: its own convergence schedule
    vs = PH.ScatterViewSet(n, 2, model="ls", dtype=torch.complex128, tol=1e-10, max_iter=200, batch=B)
    x, it = vs.solve(adjoint, torch.tensor(f, device="cuda"), torch.tensor(bs, device="cuda"))
    x = x.cpu().numpy()
    if adjoint:
        op = lambda v: v - f * G.dom_adj(v)  # noqa: E731
    else:
        op = lambda v: v - G.dom(f * v)  # noqa: E731
    for b in range(B):
        xr, itr, _ = P.bicgstab(op, bs[b], tol=1e-10, max_iter=200)
        assert int(it[b]) == itr, (b, int(it[b]), itr)
        assert np.linalg.norm(x[b] - xr) / np.linalg.norm(xr) < 1e-9

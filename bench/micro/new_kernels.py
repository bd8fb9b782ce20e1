"""Round-2 kernels at 128^3 for ncu launch lists (DRAM bytes per launch):
z-slab passes + control, standalone TV stencils, bq_wpm_phi, the resident
BQNPM metric / v_k step.  python bench/micro/new_kernels.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import _abi, slab_prox as SP, tv_ops as T, wpm as W  # noqa: E402
from paper_2307_02043_b200.configs import config2_inputs  # noqa: E402

dev = torch.device("cuda", 0)
n = 128
N = n ** 3
inp = config2_inputs(n)
f32 = torch.float32
v = torch.tensor(inp["v"], dtype=f32, device=dev)
w = W.DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=f32, device=dev),
                      d=torch.tensor(inp["d"], dtype=f32, device=dev))
g = bq.Grid((n, n, n))
# z-slab passes: 4 slabs in one process, 5 FGP iterations
sp = SP.ShardedProx(g, v, w, 0.05, W.BoxSet(0.0, np.inf), slabs_per_rank=4)
sp.run(eps=1e-300, max_iter=5)
# stencils
p = torch.randn(3, N, dtype=f32, device=dev)
for _ in range(2):
    T.gradient_stack(g, v)
    T.dual_divergence(g, p)
    T.project_dual(p, "iso")
# phi at rank 4
U4 = torch.randn(N, 4, dtype=f32, device=dev) / np.sqrt(N)
w4 = W.DiagPlusLowRank(1.25, U4)
for _ in range(2):
    W.newton_matrix(np.zeros(4), v, w4, W.BoxSet(0.0, np.inf))
# resident metric / v_k (K_s = 4 slots)
ks = 4
X = torch.randn(ks, N, dtype=f32, device=dev)
G = torch.randn(ks, N, dtype=f32, device=dev)
Us = torch.randn(ks, N, dtype=f32, device=dev) / np.sqrt(N)
EST = torch.zeros(ks, 16, dtype=torch.float64, device=dev)
EST[:, 0] = 1.0
EST[:, 1] = 1.0
meta = torch.zeros(128, dtype=torch.float64, device=dev)
Uc, acc, out = torch.empty(ks, N, dtype=f32, device=dev), torch.empty(N, dtype=f32, device=dev), torch.empty(N, dtype=f32, device=dev)
lib = _abi.load_library()
for _ in range(2):
    _abi.check(lib.bq_bqnpm_metric_vk(_abi.ctx_for(dev), _abi.BQ_F32, N, ks, _abi.ptr_array(list(X)),
                                      _abi.ptr_array(list(G)), _abi.ptr_array(list(Us)), _abi.ptr_array(list(EST)),
                                      1.0, Uc.data_ptr(), meta.data_ptr(), acc.data_ptr(), out.data_ptr(),
                                      _abi.stream_ptr(dev)), "metric_vk")
torch.cuda.synchronize()
print("ok")

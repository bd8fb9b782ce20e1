"""Host <-> device conversion helpers shared by the reference-facing mirrors.

The mirrors accept what the reference accepts (numpy arrays, Python
sequences) and additionally torch tensors.  numpy in -> numpy out keeps the
reference's ownership contract (fresh arrays out, inputs never mutated);
CUDA tensors in -> CUDA tensors out keeps GPU-resident callers free of host
round trips.
"""

from __future__ import annotations

import numpy as np
import torch


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2307_02043_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_dev(x, dtype=torch.float64, device=None, copy=False) -> torch.Tensor:
    """Contiguous device tensor of ``dtype`` (always a copy when ``copy``)."""
    device = device or default_device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=dtype)
        if copy and t.data_ptr() == x.data_ptr():
            t = t.clone()
        return t.contiguous()
    a = np.asarray(x, dtype=np.float64 if dtype == torch.float64 else np.float32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def out_like(ref, t: torch.Tensor):
    """Return ``t`` in the caller's flavour (numpy when the input was not torch)."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.detach().cpu().numpy().astype(np.float64, copy=False)


def pick_dtype(*xs, default=torch.float64) -> torch.dtype:
    for x in xs:
        if isinstance(x, torch.Tensor) and x.dtype in (torch.float32, torch.float64):
            return x.dtype
    return default

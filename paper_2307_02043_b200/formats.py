"""On-disk formats of the reference harness:
the TVQNVOL1 volume and the "tvqn-trace v1" CSV
(``/root/reference/pkg/src/tvqn/experiment_cli.py:35-137``).

Byte-compatible with the reference: a 32-byte little-endian header (magic
``TVQNVOL1``, ndim, three side lengths, 8 pad bytes) and float64 voxels in the
flat Fortran order, which is also this package's device layout -- a device
volume is written with ONE device-to-host copy and no reordering, and read
back to the device the same way.
"""

from __future__ import annotations

import csv
import struct

import numpy as np
import torch

from .solvers import IterationTrace, TraceRow

TRACE_SCHEMA = "tvqn-trace v1"
TRACE_COLUMNS = ("iter", "cost", "snr_db", "elapsed_s", "inner_iters", "grad_evals", "full_grad_evals")
VOLUME_MAGIC = b"TVQNVOL1"
_HEADER = struct.Struct("<8sI3I8x")


def _flat_and_dims(x, dims):
    if isinstance(x, torch.Tensor):
        flat = x.detach().reshape(-1).to(dtype=torch.float64, device="cpu").numpy()
        if dims is None:
            if x.ndim not in (1, 2, 3):
                raise ValueError("volumes must be 1-, 2- or 3-dimensional")
            # a C-order device tensor of shape dims[::-1] is the flat Fortran vector over dims
            dims = tuple(x.shape[::-1]) if x.ndim > 1 else (x.numel(),)
        return flat, tuple(int(k) for k in dims)
    a = np.asarray(x, dtype=float)
    if dims is not None:  # flat vector in the reference's order with explicit side lengths
        return a.reshape(-1), tuple(int(k) for k in dims)
    if not 1 <= a.ndim <= 3:
        raise ValueError("volumes must be 1-, 2- or 3-dimensional")
    return a.reshape(-1, order="F"), tuple(a.shape)


def dump_volume(x, path, dims=None):
    """Write a volume (numpy n-d array as the reference takes it, a flat vector
    with `dims`, or a device tensor)."""
    flat, dims = _flat_and_dims(x, dims)
    if not 1 <= len(dims) <= 3 or int(np.prod(dims)) != flat.size:
        raise ValueError(f"bad volume dims {dims} for {flat.size} voxels")
    header = _HEADER.pack(VOLUME_MAGIC, len(dims), *(list(dims) + [1] * (3 - len(dims))))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(flat, dtype="<f8").tobytes())


def load_volume(path, device=None):
    """Read a TVQNVOL1 file: an n-d numpy array (the reference's return), or with
    `device` the flat Fortran-order vector as a float64 device tensor."""
    with open(path, "rb") as fh:
        header = fh.read(_HEADER.size)
        if len(header) < _HEADER.size:
            raise ValueError(f"{path}: truncated header")
        magic, ndim, k1, k2, k3 = _HEADER.unpack(header)
        if magic != VOLUME_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}")
        if not 1 <= ndim <= 3:
            raise ValueError(f"{path}: bad dimensionality {ndim}")
        dims = (k1, k2, k3)[:ndim]
        count = int(np.prod(dims))
        payload = fh.read(count * 8 + 1)
        if len(payload) != count * 8:
            raise ValueError(f"{path}: payload size mismatch")
    flat = np.frombuffer(payload, dtype="<f8").copy()
    if device is not None:
        return torch.from_numpy(flat).to(device)
    return flat.reshape(dims, order="F")


def write_trace(trace: IterationTrace, path):
    """The versioned trace CSV (17 significant digits for cost and SNR)."""
    with open(path, "w", newline="") as fh:
        fh.write(f"# {TRACE_SCHEMA}\n# solver: {trace.solver}\n")
        w = csv.writer(fh)
        w.writerow(TRACE_COLUMNS)
        for r in trace.rows:
            w.writerow([r.iteration, format(r.cost, ".17g"), format(r.snr_db, ".17g"), format(r.elapsed_s, ".6f"),
                        r.inner_iters, r.grad_evals, r.full_grad_evals])


def load_trace(path) -> IterationTrace:
    with open(path, newline="") as fh:
        first = fh.readline().strip()
        if first != f"# {TRACE_SCHEMA}":
            raise ValueError(f"{path}: unsupported trace schema {first!r}")
        solver = "unknown"
        pos = fh.tell()
        line = fh.readline()
        if line.startswith("# solver:"):
            solver = line.split(":", 1)[1].strip()
        else:
            fh.seek(pos)
        rows = csv.reader(fh)
        if tuple(next(rows)) != TRACE_COLUMNS:
            raise ValueError(f"{path}: unexpected columns")
        tr = IterationTrace(solver=solver)
        for r in rows:
            tr.rows.append(TraceRow(iteration=int(r[0]), cost=float(r[1]), snr_db=float(r[2]), elapsed_s=float(r[3]),
                                    inner_iters=int(r[4]), grad_evals=int(r[5]), full_grad_evals=int(r[6])))
    return tr


__all__ = ["TRACE_SCHEMA", "TRACE_COLUMNS", "dump_volume", "load_volume", "write_trace", "load_trace"]

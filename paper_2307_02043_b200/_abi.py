"""ctypes binding of ``libbq.so`` (the C ABI declared in ``include/bq.h``).

This is the only place that knows the C signatures.  Device buffers are
passed as ``tensor.data_ptr()`` and streams as the raw ``cudaStream_t`` of
the caller's current torch stream.  A missing library or a non-B200 device
raises immediately: there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libbq.so"

BQ_OK = 0
BQ_EINVAL = -1
BQ_ECUDA = -2
BQ_ENOTPD = -3
BQ_ETIMEOUT = -4
BQ_F32 = 0
BQ_F64 = 1
BQ_TV_ISO = 0
BQ_TV_ANISO = 1
BQ_MAX_RANK = 8

# every symbol include/bq.h declares (tests check the library exports them all)
EXPORTS = (
    "bq_ctx_create",
    "bq_ctx_destroy",
    "bq_last_error",
    "bq_version",
    "bq_wtv_prox",
    "bq_wpm_box",
    "bq_metric_gram",
    "bq_metric_apply",
    "bq_dot",
    "bq_sr1",
    "bq_vk",
    "bq_tv_value",
    "bq_dct_axis",
    "bq_smooth_axis",
    "bq_views_combine",
    "bq_pointwise",
    "bq_green_init",
    "bq_ls_incident",
    "bq_ls_conv",
    "bq_ls_bicgstab",
    "bq_ls_bicgstab_small_bytes",
    "bq_ls_grad_accum",
    "bq_ls_potential",
    "bq_cscale_real",
    "bq_slab_div",
    "bq_slab_newton",
    "bq_slab_q",
    "bq_slab_dual",
    "bq_tv_diff",
    "bq_tv_grad_stack",
    "bq_tv_divergence",
    "bq_tv_project_dual",
    "bq_wpm_phi",
    "bq_bqnpm_metric_vk",
    "bq_slab_ctl",
    "bq_metric_check",
)


class WtvDesc(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("dtype", C.c_int32),
        ("dims", C.c_int64 * 3),
        ("mode", C.c_int32),
        ("rank", C.c_int32),
        ("sign", C.c_int32),
        ("accelerated", C.c_int32),
        ("tau", C.c_double),
        ("reg", C.c_double),
        ("step", C.c_double),
        ("eps", C.c_double),
        ("max_iter", C.c_int32),
        ("newton_max_iter", C.c_int32),
        ("newton_eps", C.c_double),
        ("lo", C.c_double),
        ("hi", C.c_double),
        ("lo_arr", C.c_void_p),
        ("hi_arr", C.c_void_p),
        ("d", C.c_void_p),
        ("U", C.c_void_p),
        ("v", C.c_void_p),
        ("p", C.c_void_p),
        ("pb", C.c_void_p),
        ("a", C.c_void_p),
        ("x", C.c_void_p),
        ("beta", C.c_void_p),
        ("report", C.c_void_p),
        ("p2", C.c_void_p),
        ("a2", C.c_void_p),
        ("dev_metric", C.c_void_p),
    ]


class WtvReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("newton_iterations", C.c_int32),
        ("status", C.c_int32),
        ("rel_change", C.c_double),
        ("newton_residual", C.c_double),
        ("last_newton_iterations", C.c_int32),
        ("last_newton_converged", C.c_int32),
        ("phase_ns", C.c_double * 6),
        ("phase_count", C.c_int32 * 6),
        ("phase_work_ns", C.c_double * 6),
    ]


REPORT_BYTES = C.sizeof(WtvReport)


class SlabDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32),
        ("mode", C.c_int32),
        ("rank", C.c_int32),
        ("sign", C.c_int32),
        ("K1", C.c_int64),
        ("K2", C.c_int64),
        ("L", C.c_int64),
        ("first", C.c_int32),
        ("last", C.c_int32),
        ("tau", C.c_double),
        ("reg", C.c_double),
        ("lo", C.c_double),
        ("hi", C.c_double),
        ("d", C.c_void_p),
        ("U", C.c_void_p),
        ("v", C.c_void_p),
        ("ctl", C.c_void_p),
    ]

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double

_SIGS = {
    "bq_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "bq_ctx_destroy": (C.c_int, [_P]),
    "bq_last_error": (C.c_char_p, []),
    "bq_version": (C.c_char_p, []),
    "bq_wtv_prox": (C.c_int, [_P, C.POINTER(WtvDesc), _P]),
    "bq_wpm_box": (
        C.c_int,
        [_P, _I32, _I64, _I32, _I32, _D, _P, _P, _P, _D, _D, _P, _P, _P, _D, _I32, _P, _P, _P, _P],
    ),
    "bq_metric_gram": (C.c_int, [_P, _I32, _I64, _I32, _D, _P, _P, _P, _P]),
    "bq_metric_apply": (C.c_int, [_P, _I32, _I64, _I32, _I32, _D, _P, _P, _P, _I32, _P, _P, _P]),
    "bq_dot": (C.c_int, [_P, _I32, _I64, _I32, C.POINTER(_P), C.POINTER(_P), _P, _P]),
    "bq_sr1": (C.c_int, [_P, _I32, _I64, _P, _P, _D, _D, _P, _P, _P]),
    "bq_vk": (
        C.c_int,
        [_P, _I32, _I64, _I32, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_D), _D,
         _I32, _I32, _D, _P, _P, _P, _P, _P],
    ),
    "bq_tv_value": (C.c_int, [_P, _I32, _I32, C.POINTER(_I64), _I32, _P, _P, _P]),
    "bq_dct_axis": (C.c_int, [_P, _I32, C.POINTER(_I64), _I32, _I32, _P, _P, _P]),
    "bq_smooth_axis": (C.c_int, [_P, _I32, C.POINTER(_I64), _I32, _P, _P, _P]),
    "bq_views_combine": (C.c_int, [_P, _I32, _I64, _P, C.POINTER(_P), _P, _P, _I32, _D, _P, _P, _P]),
    "bq_pointwise": (C.c_int, [_P, _I32, _I32, _I64, _P, _P, _P, _D, _P, _P]),
    "bq_green_init": (C.c_int, [_P, _I32, _I32, _D, _D, _P, _P]),
    "bq_ls_incident": (C.c_int, [_P, _I32, _I32, _D, _I32, _P, _P, _P]),
    "bq_ls_conv": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _P, _D, _D, _P, _P, _P, _P]),
    "bq_ls_bicgstab": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _D, _I32, _P, _P, _P, _P, _P]),
    "bq_ls_bicgstab_small_bytes": (C.c_int64, [_P, _I32, _I32]),
    "bq_cscale_real": (C.c_int, [_P, _I32, _I64, _I32, _P, _P, _P, _P]),
    "bq_ls_grad_accum": (C.c_int, [_P, _I32, _I64, _I32, _P, _P, _P, _D, _P, _I32, _P]),
    "bq_ls_potential": (C.c_int, [_P, _I32, _I64, _P, _D, _D, _I32, _P, _P, _P]),
    "bq_slab_div": (C.c_int, [_P, C.POINTER(SlabDesc), _P, _P, _P, _P, _P]),
    "bq_slab_newton": (C.c_int, [_P, C.POINTER(SlabDesc), _P, C.POINTER(_D), C.POINTER(_D), _P, _P]),
    "bq_slab_q": (C.c_int, [_P, C.POINTER(SlabDesc), _P, C.POINTER(_D), C.POINTER(_D), _P, _P]),
    "bq_metric_check": (C.c_int, [_P, _I32, _I64, _I32, _P, _P, _P, _P]),
    "bq_slab_ctl": (C.c_int, [_P, C.POINTER(SlabDesc), _I32, _P, _D, _I32, _D, _P]),
    "bq_slab_dual": (C.c_int, [_P, C.POINTER(SlabDesc), _P, _P, _P, _P, _D, _D, _P, _P, _P, _P]),
    "bq_tv_diff": (C.c_int, [_P, _I32, _I32, C.POINTER(_I64), _I32, _I32, _P, _P, _P]),
    "bq_tv_grad_stack": (C.c_int, [_P, _I32, _I32, C.POINTER(_I64), _P, _P, _P]),
    "bq_tv_divergence": (C.c_int, [_P, _I32, _I32, C.POINTER(_I64), _P, _P, _P]),
    "bq_tv_project_dual": (C.c_int, [_P, _I32, _I32, _I64, _I32, _P, _P, _P]),
    "bq_bqnpm_metric_vk": (C.c_int, [_P, _I32, _I64, _I32, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                     C.POINTER(_P), _D, _P, _P, _P, _P, _P]),
    "bq_wpm_phi": (C.c_int, [_P, _I32, _I64, _I32, _I32, _D, _P, _P, _P, _D, _D, _P, _P, _P, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()
_ctx = {}


class BqError(RuntimeError):
    pass


def load_library(path: Path | str | None = None):
    """Load libbq.so and declare the signatures (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        import os

        p = Path(path) if path is not None else Path(os.environ.get("BQ_LIB") or LIB_PATH)
        if not p.exists():
            raise BqError(
                f"{p} is missing: build it with `python -m paper_2307_02043_b200.build` "
                "(the product path has no CPU fallback)"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = ""):
    """Map a bq status to the reference's exception types."""
    if rc == BQ_OK:
        return
    msg = (load_library().bq_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (BQ_EINVAL, BQ_ENOTPD):
        raise ValueError(text)
    raise BqError(f"{text} (status {rc})")


def ctx_for(device: torch.device | int | None = None) -> int:
    """Per-(device, thread) context handle, created on first use."""
    if not torch.cuda.is_available():
        raise BqError("a CUDA device is required: libbq has no CPU path")
    if device is None:
        idx = torch.cuda.current_device()
    elif isinstance(device, torch.device):
        idx = device.index if device.index is not None else torch.cuda.current_device()
    else:
        idx = int(device)
    key = (idx, threading.get_ident())
    h = _ctx.get(key)
    if h is None:
        lib = load_library()
        out = C.c_void_p()
        with torch.cuda.device(idx):
            check(lib.bq_ctx_create(idx, C.byref(out)), "bq_ctx_create")
        h = out.value
        _ctx[key] = h
    return h


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return BQ_F32
    if dt == torch.float64:
        return BQ_F64
    raise ValueError(f"unsupported dtype {dt}: libbq computes in float32 or float64")


def ptr_array(tensors):
    arr = (C.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr

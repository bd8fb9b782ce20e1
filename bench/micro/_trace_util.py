"""Locate the trace buffer (the stream workspace's device scratch) of a context.

bq_ctx: {int device, num_sms; void* fft_cache; StreamWs* streams[16]; int n_streams};
StreamWs: {cudaStream_t stream; Workspace{partials, barrier, ctl, ctl_bytes, scratch}; ...}."""
import ctypes

import torch


def trace_scratch(ctx, warm):
    """`warm()` must have launched on the current stream once (the workspace is created on first use)."""
    warm()
    torch.cuda.synchronize()
    raw = ctypes.cast(ctx, ctypes.POINTER(ctypes.c_uint64))
    n = ctypes.cast(ctx, ctypes.POINTER(ctypes.c_int32))[2 * 18]
    cur = torch.cuda.current_stream().cuda_stream
    for i in range(n):
        sw = ctypes.cast(ctypes.c_void_p(raw[2 + i]), ctypes.POINTER(ctypes.c_uint64))
        if sw[0] == cur:
            return sw[5]
    raise RuntimeError("no workspace for the current stream")

"""Helpers for GPU parity tests: run one node operator through the C ABI
(hs_launch) on torch-allocated device memory, and compare with the oracle."""
from __future__ import annotations

import ctypes

import numpy as np

from paper_2009_07482_b200 import _native

OPS = {"gemm": 0, "gemm_nt": 1, "gemm_relu": 2, "transpose": 3, "scale": 4, "softmax": 5, "add": 6,
       "add_layernorm": 7, "concat": 8, "attn_head": 9, "head": 10}
MATH = {"tf32x3": 0, "tf32": 1, "simt": 2, "bf16x3": 3}

_ctx = None
_stream = None


def stream():
    global _ctx, _stream
    L = _native.lib()
    if _stream is None:
        ctx = ctypes.c_void_p()
        _native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
        s = ctypes.c_void_p()
        _native.check(L.hs_stream_create(ctx, 0, ctypes.byref(s)))
        _ctx, _stream = ctx, s
    return _stream


def split_weights(B, transposed, N, K, bf16=False):
    """Pre-split a shared GEMM B into K-major hi/lo planes (tf32, or bf16 for math bf16x3)."""
    import torch
    planes = torch.empty(2 * N * K, device="cuda")  # fp32-sized: bf16 planes use half of it
    torch.cuda.synchronize()  # B was produced on torch's stream
    L = _native.lib()
    _native.check(L.hs_gemm_split_weights_ex(stream(), B.data_ptr(), int(transposed), N, K, planes.data_ptr(), N * K,
                                             int(bf16)))
    _native.check(L.hs_stream_sync(stream()))
    return planes


def launch(op, inputs, out, dims, fparam=(1.0, 1e-5), math="tf32x3", batch=1, strides=None, out_stride=None,
           aux=None, out_ld=0, epilogue=0, out_offset=0):
    """inputs/out: torch CUDA float32 tensors shaped [batch, elems] or [elems] (shared).
    out_offset (elements) / out_ld / epilogue: GEMM output placement and epilogue."""
    import torch
    # Our stream is non-blocking: it does not order after torch's stream, so the
    # tensors torch just filled/copied must be complete before we launch.
    torch.cuda.synchronize()
    L = _native.lib()
    a = _native.OpArgs()
    a.out_ld = out_ld
    a.epilogue = epilogue
    a.aux = aux.data_ptr() if aux is not None else None
    a.n_in = len(inputs)
    for i, t in enumerate(inputs):
        a.in_[i] = t.data_ptr()
        a.in_stride[i] = (strides[i] if strides else (0 if t.dim() == 1 else t.shape[-1]))
    a.out = out.data_ptr() + 4 * out_offset
    a.out_stride = out_stride if out_stride is not None else out.shape[-1]
    for i, d in enumerate(dims):
        a.dims[i] = d
    a.fparam[0], a.fparam[1] = fparam
    _native.check(L.hs_launch(stream(), OPS[op], ctypes.byref(a), MATH[math], batch), f"hs_launch({op})")
    _native.check(L.hs_stream_sync(stream()), "sync")


def normwise(y, ref):
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))

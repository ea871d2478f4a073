"""GEMM microbenchmark through hs_launch: per-launch device time for the
config shapes under several variants (math, batch, K, pre-split B)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402

L = _native.lib()
ctx, st, e0, e1 = (ctypes.c_void_p() for _ in range(4))
_native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
_native.check(L.hs_stream_create(ctx, 0, ctypes.byref(st)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))
OPS = {"gemm": 0, "gemm_nt": 1, "gemm_relu": 2}
MATH = {"tf32x3": 0, "tf32": 1, "simt": 2}


def run(M, N, K, batch, op="gemm", math="tf32x3", presplit=True, shared=True, reps=20):
    A = torch.randn(batch, M * K, device="cuda")
    B = torch.randn(N * K if shared else batch * N * K, device="cuda")
    C = torch.empty(batch, M * N, device="cuda")
    planes = None
    if presplit and shared:
        planes = torch.empty(2 * N * K, device="cuda")
        _native.check(L.hs_gemm_split_weights(st, B.data_ptr(), int(op == "gemm_nt"), N, K, planes.data_ptr()))
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0 if shared else N * K
    a.out, a.out_stride = C.data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr() if planes is not None else None
    for _ in range(3):
        _native.check(L.hs_launch(st, OPS[op], ctypes.byref(a), MATH[math], batch))
    _native.check(L.hs_stream_sync(st))
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        _native.check(L.hs_launch(st, OPS[op], ctypes.byref(a), MATH[math], batch))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    us = ns.value / 1e3 / reps
    flops = 2.0 * M * N * K * batch
    print(f"{op:9s} M={M:4d} N={N:5d} K={K:5d} batch={batch:4d} math={math:6s} presplit={int(presplit)} "
          f"shared={int(shared)}: {us:8.2f} us  {flops / us / 1e6:7.1f} TFLOP/s", flush=True)
    return us


if __name__ == "__main__":
    for batch in (64, 128, 148, 296, 592):
        run(128, 64, 512, batch)
    for K in (128, 512, 2048):
        run(128, 64, K, 148)
    run(128, 64, 512, 148, math="tf32")
    run(128, 64, 512, 148, presplit=False)
    run(128, 64, 64, 128)
    run(128, 64, 128, 128, shared=False, presplit=False)
    run(128, 128, 64, 128, shared=False, presplit=False)
    for batch in (64, 128, 256):
        run(128, 2048, 512, batch, op="gemm_relu")
        run(128, 512, 2048, batch)
    run(128, 2048, 512, 128, op="gemm_relu", math="tf32")

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


def run(M, N, K, batch, op="gemm", math="tf32x3", presplit=True, shared=True, reps=20, epilogue=0, fill=None):
    A = torch.randn(batch, M * K, device="cuda")
    B = torch.randn(N * K if shared else batch * N * K, device="cuda")
    if fill is not None:  # operand values for data-dependent power experiments ("zeros", "ones")
        v = {"zeros": 0.0, "ones": 1.0}[fill]
        A.fill_(v)
        B.fill_(v)
    C = torch.empty(batch, M * N, device="cuda")
    planes = None
    if presplit and shared:
        planes = torch.empty(2 * N * K, device="cuda")
        _native.check(L.hs_gemm_split_weights(st, B.data_ptr(), int(op == "gemm_nt"), N, K, planes.data_ptr()))
    torch.cuda.synchronize()
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0 if shared else N * K
    a.out, a.out_stride = C.data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr() if planes is not None else None
    a.epilogue = epilogue
    a.fparam[0] = 0.125
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
          f"shared={int(shared)} epi={epilogue}: {us:8.2f} us  {flops / us / 1e6:7.1f} TFLOP/s", flush=True)
    return us


def run_grouped(M, N, K, batch, members=3, reps=20):
    """Grouped launch: `members` sibling GEMMs sharing A, N columns each, one launch."""
    A = torch.randn(batch, M * K, device="cuda")
    Bs = [torch.randn(N * K, device="cuda") for _ in range(members)]
    planes = torch.empty(2 * members * N * K, device="cuda")
    for m, B in enumerate(Bs):
        _native.check(L.hs_gemm_split_weights_strided(st, B.data_ptr(), 0, N, K, planes.data_ptr() + 4 * m * N * K,
                                                      members * N * K))
    Cs = [torch.empty(batch, M * N, device="cuda") for _ in range(members)]
    torch.cuda.synchronize()
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), Bs[0].data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0
    a.out, a.out_stride = Cs[0].data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr()
    a.n_out = members
    for m in range(members):
        a.outs[m], a.out_strides[m] = Cs[m].data_ptr(), M * N
    for _ in range(3):
        _native.check(L.hs_launch(st, 0, ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        _native.check(L.hs_launch(st, 0, ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    us = ns.value / 1e3 / reps
    flops = 2.0 * M * N * K * batch * members
    print(f"grouped   M={M:4d} N={members}x{N:3d} K={K:5d} batch={batch:4d}: {us:8.2f} us  {flops / us / 1e6:7.1f} TFLOP/s",
          flush=True)


if __name__ == "__main__":
    for batch in (128, 148, 256):
        run_grouped(128, 64, 512, batch)
    run_grouped(128, 64, 512, 128, members=2)
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

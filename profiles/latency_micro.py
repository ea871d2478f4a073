"""Per-launch fixed cost of node kernels: back-to-back stream launches vs the
same launches captured in a CUDA graph (hs_capture_*), for a 1-K-block GEMM,
a small elementwise add and a softmax."""
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


def timed(fn, reps=50, graph=False):
    for _ in range(3):
        fn()
    _native.check(L.hs_stream_sync(st))
    g = None
    if graph:
        g = ctypes.c_void_p()
        _native.check(L.hs_capture_begin(st))
        for _ in range(reps):
            fn()
        _native.check(L.hs_capture_end(st, ctypes.byref(g)))
        _native.check(L.hs_graph_launch(g, st))
        _native.check(L.hs_stream_sync(st))
    _native.check(L.hs_event_record(e0, st))
    if graph:
        _native.check(L.hs_graph_launch(g, st))
    else:
        for _ in range(reps):
            fn()
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    if g is not None:
        L.hs_graph_destroy(g)
    return ns.value / 1e3 / reps


def gemm_fn(M, N, K, batch):
    A = torch.randn(batch, M * K, device="cuda")
    B = torch.randn(N * K, device="cuda")
    C = torch.empty(batch, M * N, device="cuda")
    planes = torch.empty(2 * N * K, device="cuda")
    _native.check(L.hs_gemm_split_weights(st, B.data_ptr(), 0, N, K, planes.data_ptr()))
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0
    a.out, a.out_stride = C.data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr()
    keep = (A, B, C, planes)
    return lambda: (keep, _native.check(L.hs_launch(st, 0, ctypes.byref(a), 0, batch)))


def op_fn(op, n, batch, dims, fparam=(1.0, 1e-5)):
    A = torch.randn(batch, n, device="cuda")
    B = torch.randn(batch, n, device="cuda")
    C = torch.empty(batch, n, device="cuda")
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr()
    a.in_stride[0], a.in_stride[1] = n, n
    a.out, a.out_stride = C.data_ptr(), n
    for i, d in enumerate(dims):
        a.dims[i] = d
    a.fparam[0], a.fparam[1] = fparam
    keep = (A, B, C)
    return lambda: (keep, _native.check(L.hs_launch(st, op, ctypes.byref(a), 0, batch)))


cases = {
    "gemm 128x64x32 batch=1 (1 CTA, 1 K-block)": gemm_fn(128, 64, 32, 1),
    "gemm 128x64x32 batch=148": gemm_fn(128, 64, 32, 148),
    "gemm 128x64x512 batch=1": gemm_fn(128, 64, 512, 1),
    "gemm 128x64x512 batch=128": gemm_fn(128, 64, 512, 128),
    "add n=256 batch=1": op_fn(6, 256, 1, [256]),
    "add n=65536 batch=128": op_fn(6, 65536, 128, [65536]),
    "softmax 128x128 batch=128": op_fn(5, 16384, 128, [128, 128], (0.125, 1e-5)),
}
for name, fn in cases.items():
    s = timed(fn)
    g = timed(fn, graph=True)
    print(f"{name:45s} stream {s:7.2f} us/launch   graph {g:7.2f} us/node", flush=True)

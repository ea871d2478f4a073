"""Per-launch fixed cost of node kernels inside CUDA graphs (hs_capture_*):
GEMMs of 1 and 16 K-blocks with 1 and 148 CTAs, and small HBM-bound nodes.
Back-to-back stream launches from Python are host-bound for small kernels, so
graph replay is the number that matters for the engine."""
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


def graph_us(fn, reps=50):
    fn()
    _native.check(L.hs_stream_sync(st))
    g = ctypes.c_void_p()
    _native.check(L.hs_capture_begin(st))
    for _ in range(reps):
        fn()
    _native.check(L.hs_capture_end(st, ctypes.byref(g)))
    for _ in range(2):
        _native.check(L.hs_graph_launch(g, st))
    _native.check(L.hs_stream_sync(st))
    _native.check(L.hs_event_record(e0, st))
    _native.check(L.hs_graph_launch(g, st))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    L.hs_graph_destroy(g)
    return ns.value / 1e3 / reps


def gemm_fn(M, N, K, batch, shared=True):
    A = torch.randn(batch, M * K, device="cuda")
    B = torch.randn(N * K if shared else batch * N * K, device="cuda")
    C = torch.empty(batch, M * N, device="cuda")
    planes = None
    if shared:
        planes = torch.empty(2 * N * K, device="cuda")
        _native.check(L.hs_gemm_split_weights(st, B.data_ptr(), 0, N, K, planes.data_ptr()))
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0 if shared else N * K
    a.out, a.out_stride = C.data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr() if planes is not None else None
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


CASES = {
    "gemm 128x64x32 batch=1": lambda: gemm_fn(128, 64, 32, 1),
    "gemm 128x64x32 batch=148": lambda: gemm_fn(128, 64, 32, 148),
    "gemm 128x64x512 batch=1": lambda: gemm_fn(128, 64, 512, 1),
    "gemm 128x64x512 batch=148": lambda: gemm_fn(128, 64, 512, 148),
    "gemm 128x128x512 batch=148": lambda: gemm_fn(128, 128, 512, 148),
    "dag QK^T 128x128x64 act-B batch=256": lambda: gemm_fn(128, 128, 64, 256, shared=False),
    "dag PV 128x64x128 act-B batch=256": lambda: gemm_fn(128, 64, 128, 256, shared=False),
    "dag CW 128x64x64 weight batch=256": lambda: gemm_fn(128, 64, 64, 256),
    "dag FFN2 128x512x2048 batch=256": lambda: gemm_fn(128, 512, 2048, 256),
    "add n=256 batch=1": lambda: op_fn(6, 256, 1, [256]),
    "softmax 128x128 batch=128": lambda: op_fn(5, 16384, 128, [128, 128], (0.125, 1e-5)),
}

if __name__ == "__main__":
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for name, make in CASES.items():
        if only and only not in name:
            continue
        print(f"{name:32s} graph {graph_us(make()):7.2f} us/node", flush=True)

"""Fused attention head (HS_OP_ATTN_HEAD) vs the unfused tcgen05 chain it replaces
(gemm_nt+softmax epilogue -> gemm P·V -> gemm C·W), 128x64 heads, batch 256."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402
from tests.gpu_util import split_weights, stream  # noqa: E402

L = _native.lib()
S, dk, batch = 128, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 256
Q, K, V = (torch.randn(batch, S * dk, device="cuda") for _ in range(3))
W = torch.randn(dk * dk, device="cuda") / 8
planes = split_weights(W, False, dk, dk)
P = torch.empty(batch, S * S, device="cuda")
C = torch.empty(batch, S * dk, device="cuda")
Z = torch.empty(batch, S * dk, device="cuda")
torch.cuda.synchronize()
st = stream()


def args(op_in, out, dims, aux=None, epi=0):
    a = _native.OpArgs()
    a.n_in = len(op_in)
    for i, t in enumerate(op_in):
        a.in_[i] = t.data_ptr()
        a.in_stride[i] = 0 if t.dim() == 1 else t.shape[-1]
    a.out, a.out_stride = out.data_ptr(), out.shape[-1]
    for i, d in enumerate(dims):
        a.dims[i] = d
    a.fparam[0] = 0.125
    a.aux = aux.data_ptr() if aux is not None else None
    a.epilogue = epi
    return a


chain = [(1, args([Q, K], P, [S, S, dk], epi=1)), (0, args([P, V], C, [S, dk, S])),
         (0, args([C, W], Z, [S, dk, dk], aux=planes))]
fused = [(9, args([Q, K, V, W], Z, [S, dk, dk], aux=planes))]
ctx = ctypes.c_void_p()
_native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))
for name, seq in (("unfused chain", chain), ("attn_head", fused)):
    for _ in range(3):
        for op, a in seq:
            _native.check(L.hs_launch(st, op, ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e0, st))
    reps = 20
    for _ in range(reps):
        for op, a in seq:
            _native.check(L.hs_launch(st, op, ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    print(f"{name:14s} batch={batch}: {ns.value / 1e3 / reps:8.2f} us per head-batch", flush=True)

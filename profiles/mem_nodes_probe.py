"""The HBM-bound node kernels (add, scale, softmax, transpose, concat, add+LayerNorm) at
batch sizes far above L2, launched through hs_launch, for an ncu metrics pass:
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python profiles/mem_nodes_probe.py
Also prints event-timed GB/s (algorithmic bytes) per op."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402
from tests.gpu_util import OPS, stream  # noqa: E402

L = _native.lib()
st = stream()
ctx, e0, e1 = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
_native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))
R, C, batch = 128, 512, 1024  # one encoder activation per instance (256 KB), 256 MB per operand
n = R * C


def run(name, ins, out, dims, nbytes, fparam=(1.0, 1e-5), reps=10):
    a = _native.OpArgs()
    a.n_in = len(ins)
    for i, t in enumerate(ins):
        a.in_[i] = t.data_ptr()
        a.in_stride[i] = 0 if t.dim() == 1 else t.shape[-1]
    a.out, a.out_stride = out.data_ptr(), out.shape[-1]
    for i, d in enumerate(dims):
        a.dims[i] = d
    a.fparam[0], a.fparam[1] = fparam
    torch.cuda.synchronize()
    for _ in range(2):
        _native.check(L.hs_launch(st, OPS[name], ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        _native.check(L.hs_launch(st, OPS[name], ctypes.byref(a), 0, batch))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    t = ns.value / 1e9 / reps
    print(f"{name:14s} {t * 1e6:8.1f} us  {nbytes / t / 1e9:7.0f} GB/s (algorithmic {nbytes / 1e6:.0f} MB)", flush=True)


A, B, Y = (torch.randn(batch, n, device="cuda") for _ in range(3))
g, be = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
run("add", [A, B], Y, [n], batch * 3 * n * 4)
run("scale", [A], Y, [n], batch * 2 * n * 4, fparam=(0.125, 1e-5))
S = 128
P = torch.randn(batch, S * S * 4, device="cuda")  # four 128x128 score blocks per instance
Q = torch.empty_like(P)
run("softmax", [P], Q, [4 * S, S], batch * 2 * 4 * S * S * 4, fparam=(0.125, 1e-5))
run("transpose", [A], Y, [R, C], batch * 2 * n * 4)
Z = [torch.randn(batch, R * 64, device="cuda") for _ in range(8)]
run("concat", Z, Y, [R, 64], batch * 2 * n * 4)
run("add_layernorm", [A, B, g, be], Y, [R, C], batch * 3 * n * 4 + 8 * C)

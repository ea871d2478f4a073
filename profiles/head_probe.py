"""Whole-head kernel (HS_OP_HEAD: Q/K/V projection + attention in one CTA-pair launch)
vs the two launches it replaces (grouped Q/K/V pair GEMM -> attn_head), per batch.
usage: python profiles/head_probe.py [batch ...]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402
from tests.gpu_util import split_weights, stream  # noqa: E402
from tests.test_gpu_kernels import _grouped_qkv, _head_launch, _qkv_planes  # noqa: E402

L = _native.lib()
S, D = 128, 512
st = stream()
e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
ctx = ctypes.c_void_p()
_native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
_native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        fn()
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    return ns.value / 1e3 / reps


def attn_args(Q, K, V, Wh, ph, Z):
    a = _native.OpArgs()
    a.n_in = 4
    for i, t in enumerate((Q, K, V, Wh)):
        a.in_[i] = t.data_ptr()
        a.in_stride[i] = 0 if t.dim() == 1 else t.shape[-1]
    a.out, a.out_stride = Z.data_ptr(), Z.shape[-1]
    a.dims[0], a.dims[1], a.dims[2] = S, 64, 64
    a.fparam[0] = 0.125
    a.aux = ph.data_ptr()
    return a


for batch in [int(b) for b in sys.argv[1:]] or (64, 148, 296, 512):
    X = torch.randn(batch, S * D, device="cuda")
    Ws = [torch.randn(D * 64, device="cuda") / np.sqrt(D) for _ in range(3)]
    Wh = torch.randn(64 * 64, device="cuda") / 8
    pq, ph = _qkv_planes(Ws, D), split_weights(Wh, False, 64, 64)
    Q, K, V, Z = (torch.empty(batch, S * 64, device="cuda") for _ in range(4))
    aa = attn_args(Q, K, V, Wh, ph, Z)
    # the ABI helpers synchronise after each launch; time raw launches instead
    h = _native.OpArgs()
    h.n_in = 2
    h.in_[0], h.in_stride[0] = X.data_ptr(), S * D
    h.in_[1], h.in_stride[1] = ph.data_ptr(), 0
    h.aux = pq.data_ptr()
    h.out, h.out_stride = Z.data_ptr(), S * 64
    h.dims[0], h.dims[1], h.dims[2] = S, D, 64
    h.fparam[0] = 0.125
    g = _native.OpArgs()
    g.n_in = 2
    g.in_[0], g.in_stride[0] = X.data_ptr(), S * D
    g.in_[1], g.in_stride[1] = Ws[0].data_ptr(), 0
    g.out, g.out_stride = Q.data_ptr(), S * 64
    g.dims[0], g.dims[1], g.dims[2] = S, 64, D
    g.aux = pq.data_ptr()
    g.n_out = 3
    for m, t in enumerate((Q, K, V)):
        g.outs[m], g.out_strides[m] = t.data_ptr(), S * 64
    torch.cuda.synchronize()
    t_qkv = timed(lambda: _native.check(L.hs_launch(st, 0, ctypes.byref(g), 0, batch)))
    t_att = timed(lambda: _native.check(L.hs_launch(st, 9, ctypes.byref(aa), 0, batch)))
    t_head = timed(lambda: _native.check(L.hs_launch(st, 10, ctypes.byref(h), int(os.environ.get('HEAD_MATH', '0')), batch)))
    flops = batch * (2.0 * S * 192 * D + 2.0 * S * S * 64 * 2 + 2.0 * S * 64 * 64)
    print(f"batch={batch:4d}  grouped QKV {t_qkv:7.2f} us + attn_head {t_att:6.2f} us = {t_qkv + t_att:7.2f} us | "
          f"head {t_head:7.2f} us  ({flops / t_head / 1e6:6.1f} TFLOP/s algorithmic)", flush=True)

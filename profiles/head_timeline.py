"""Per-instance phase timeline of the whole-head kernel, CTA 0 (needs a library built
with -DHS_DBG_TIMELINE=1, e.g. variants/build.sh timeline "-DHS_DBG_TIMELINE=1" and
HETSIM_LIB=variants/lib_timeline.so). clock64 cycles relative to instance 0's start.
usage: python profiles/head_timeline.py [batch=592]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402
from tests.gpu_util import split_weights, stream  # noqa: E402
from tests.test_gpu_kernels import _qkv_planes  # noqa: E402

L = _native.lib()
S, D = 128, 512
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 592
X = torch.randn(batch, S * D, device="cuda")
Ws = [torch.randn(D * 64, device="cuda") / np.sqrt(D) for _ in range(3)]
Wh = torch.randn(64 * 64, device="cuda") / 8
pq, ph = _qkv_planes(Ws, D), split_weights(Wh, False, 64, 64)
Z = torch.empty(batch, S * 64, device="cuda")
h = _native.OpArgs()
h.n_in = 2
h.in_[0], h.in_stride[0] = X.data_ptr(), S * D
h.in_[1], h.in_stride[1] = ph.data_ptr(), 0
h.aux = pq.data_ptr()
h.out, h.out_stride = Z.data_ptr(), S * 64
h.dims[0], h.dims[1], h.dims[2] = S, D, 64
h.fparam[0] = 0.125
torch.cuda.synchronize()
for _ in range(3):
    _native.check(L.hs_launch(stream(), 10, ctypes.byref(h), 0, batch))
_native.check(L.hs_stream_sync(stream()))
assert L.hs_debug_head_timeline_reset() == 0, "library built without HS_DBG_TIMELINE"
_native.check(L.hs_launch(stream(), 10, ctypes.byref(h), 0, batch))
_native.check(L.hs_stream_sync(stream()))
buf = (ctypes.c_longlong * 256)()
L.hs_debug_head_timeline.argtypes = [ctypes.c_void_p]
assert L.hs_debug_head_timeline(ctypes.cast(buf, ctypes.c_void_p)) == 0, "library built without HS_DBG_TIMELINE"
tl = np.array(buf[:], dtype=np.int64).reshape(8, 32)
names = ["mma:proj_start", "mma:proj_issued", "att:acc_full", "att:s_full", "att:c_full", "att:z_stored"]  # slots 0-5
ext = {24: "ext:q", 25: "ext:k", 26: "ext:v_issued", 27: "ext:done_w8", 28: "ext:done_w15"}
waits = {6: "mma_wait_extpair", 7: "mma_proj_issue", 8: "mma_wait_W", 9: "mma_wait_A", 10: "conv_wait_X",
         11: "conv_wait_Aempty", 12: "xtma_wait_empty", 13: "wtma_wait_empty", 14: "conv_work", 15: "conv_signal",
         16: "att_wait_ext", 17: "att_wait_sfull", 18: "att_wait_p0", 19: "att_wait_p1", 20: "att_wait_c"}
t0 = tl[0, 0]  # stamps are the low 32 bits of clock64
per_cta = -(-batch // 148)
for t in range(min(per_cta, 8)):
    print(f"pair {t}: " + "  ".join(f"{n}={(tl[t, k] - t0) % 2**32}" for k, n in enumerate(names)))
    print("    extraction: " + "  ".join(f"{n}={(tl[t, k] - t0) % 2**32}" for k, n in ext.items()))
    print("    waits: " + "  ".join(f"{n}={tl[t, k]}" for k, n in waits.items()))

"""Where a single-instance tcgen05 GEMM spends its time: clock64 stamps of CTA 0 of
gemm_tc_kernel (library built with -DHS_DBG_GEMM_TL=1: variants/build.sh gemmtl
"-DHS_DBG_GEMM_TL=1"; HETSIM_LIB=variants/lib_gemmtl.so).
usage: python profiles/gemm_timeline.py [M N K] [deterministic=0]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native  # noqa: E402
from tests.gpu_util import launch  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (256, 256, 256)
det = int(sys.argv[4]) if len(sys.argv) > 4 else 0
L = _native.lib()
L.hs_debug_gemm_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
A = torch.randn(1, M * K, device="cuda")
B = torch.randn(1, K * N, device="cuda")
C = torch.empty(1, M * N, device="cuda")
names = ["entry", "prologue", "pdl_wait", "tma0", "conv_st_full0", "conv_op_full0", "mma_commit0", "epi_acc_full",
         "epi_done", "pre_exit_sync", "dealloc", "csplit_cta_sync", "csplit_cluster_sync", "csplit_reduced",
         "csplit_cluster_sync2"]
for rep in range(3):
    assert L.hs_debug_gemm_timeline(None, 1) == 0, "library built without HS_DBG_GEMM_TL"
    launch("gemm", [A, B], C, [M, N, K])
buf = (ctypes.c_longlong * 16)()
L.hs_debug_gemm_timeline(ctypes.cast(buf, ctypes.c_void_p), 0)
t0 = buf[0]
print(f"gemm {M}x{N}x{K}: " + "  ".join(f"{n}={buf[i] - t0}" for i, n in enumerate(names) if buf[i]))

"""Single-instance GEMM latency (the C1/C2/C3 node shapes) through hs_launch,
back-to-back launches on one stream: tf32x3 (split-K on / off) vs the CUDA-core
fp32 kernel. usage: python profiles/small_gemm.py"""
import sys

sys.path.insert(0, ".")
from profiles.gemm_micro import run  # noqa: E402

for (M, N, K, op, presplit, shared) in ((256, 256, 256, "gemm", False, False), (128, 128, 64, "gemm_nt", False, False),
                                        (128, 64, 128, "gemm", False, False), (128, 2048, 512, "gemm_relu", True, True),
                                        (128, 512, 2048, "gemm", True, True)):
    for math in ("tf32x3", "simt"):
        run(M, N, K, 1, op=op, math=math, presplit=presplit, shared=shared, reps=50)

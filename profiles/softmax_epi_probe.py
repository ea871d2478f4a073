"""QK^T (gemm_nt 128x128x64 x256) with and without the softmax epilogue, for timing and ncu."""
import sys
sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
gm.run(128, 128, 64, 256, op="gemm_nt", presplit=False, shared=False, reps=reps, epilogue=1)
gm.run(128, 128, 64, 256, op="gemm_nt", presplit=False, shared=False, reps=reps, epilogue=0)
gm.run(128, 128, 64, 256, op="gemm", presplit=False, shared=False, reps=reps, epilogue=0)

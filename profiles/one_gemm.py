"""Launch one GEMM config a few times (for focused ncu captures)."""
import sys
sys.path.insert(0, ".")
sys.argv += []
from profiles import gemm_micro as gm  # noqa: E402
M, N, K, batch = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (128, 64, 512, 148)))
gm.run(M, N, K, batch, reps=3)

"""Steady-state GEMM tile cost for the A/B variant libraries (variants/ab.sh)."""
import sys
sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402
gm.run_grouped(128, 64, 512, 592)
gm.run(128, 2048, 512, 37, op="gemm_relu")
gm.run(128, 2048, 512, 256, op="gemm_relu")
gm.run(128, 512, 2048, 256)

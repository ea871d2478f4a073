"""FFN1 / FFN2 / grouped-QKV pair GEMMs at batch 512 (bench.gemm_roofline-style timing) for A/B runs."""
import sys
sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402
gm.run(128, 2048, 512, 512, op="gemm_relu")
gm.run(128, 512, 2048, 512)

"""FFN1 / FFN2 pair GEMMs across batch sizes (for A/B of pair tile widths)."""
import sys
sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402
for batch in (64, 512):
    gm.run(128, 2048, 512, batch, op="gemm_relu")
    gm.run(128, 512, 2048, batch)

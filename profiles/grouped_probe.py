"""Per-tile cost of the grouped QKV launch (3 x 128x64x512, N=192 tiles) vs batch,
next to FFN1 (128x2048x512, N=128 tiles): separates fixed launch cost, wave
quantisation and steady-state tile cost."""
import sys
sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402
for batch in (1, 148, 296, 592):
    gm.run_grouped(128, 64, 512, batch)
for batch in (10, 19, 37):
    gm.run(128, 2048, 512, batch, op="gemm_relu")

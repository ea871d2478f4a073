"""Grouped Q/K/V projection of one head (3 x 128x64x512 per instance, one CTA-pair launch,
N=192 tiles) vs batch, and FFN1 at the same batch for reference.
usage: python profiles/qkv_probe.py [batch ...]"""
import sys

sys.path.insert(0, ".")
from profiles import gemm_micro as gm  # noqa: E402

for batch in [int(b) for b in sys.argv[1:]] or (64, 148, 296, 512, 1024):
    gm.run_grouped(128, 64, 512, batch)

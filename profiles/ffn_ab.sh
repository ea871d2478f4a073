#!/bin/bash
# A/B of the FFN pair GEMMs (FFN1 128x2048x512, FFN2 128x512x2048; batch 512, tf32x3,
# resident pre-split weights) across library variants
for L in paper_2009_07482_b200/libhetsim.so variants/lib_*.so; do
  echo "== $L"
  HETSIM_LIB=$L python - <<'PY'
import sys; sys.path.insert(0, ".")
from profiles.gemm_micro import run
run(128, 2048, 512, 512, op="gemm_relu", reps=20)
run(128, 512, 2048, 512, op="gemm", reps=20)
PY
done

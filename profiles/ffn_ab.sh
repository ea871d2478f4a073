#!/bin/bash
# A/B of the FFN pair GEMM (FFN1 and FFN2 shapes, batch 512, tf32x3) across library variants
for L in paper_2009_07482_b200/libhetsim.so variants/lib_*.so; do
  echo "== $L"
  HETSIM_LIB=$L python - <<'PY'
import sys; sys.path.insert(0, ".")
import bench
for shape in ("ffn1",):
    tf, ms, fl = bench.gemm_roofline(512, "tf32x3", reps=20)
    print(f"  ffn1 x512 {ms*1e3:.1f} us {tf:.1f} TFLOP/s")
PY
done

for L in paper_2009_07482_b200/libhetsim.so variants/lib_*.so; do
  echo "== $L"
  HETSIM_LIB=$L python -c "
import sys; sys.path.insert(0, '.')
from profiles.gemm_micro import run
run(128, 2048, 512, 512, op='gemm_relu', reps=20)
run(128, 512, 2048, 512, op='gemm', reps=20)
" 2>&1 | tail -2
done

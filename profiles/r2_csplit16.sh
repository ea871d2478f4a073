mkdir -p gpurun_out
{ HETSIM_LIB=variants/lib_cs16.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm_parity or split_k" 2>&1 | tail -2
for v in default cs16 default cs16; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib python profiles/r2_c3_fuse.py 2>&1 | head -3
done; } > gpurun_out/r2_csplit16.txt 2>&1

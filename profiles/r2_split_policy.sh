# latency configs against the split-K policy: default (cluster split, >= 1 K-block per split),
# >= 2 / >= 4 K-blocks per split, no split at all
mkdir -p gpurun_out
{ for v in default nosplit mkb2 mkb4 default nosplit; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib timeout 300 python profiles/r2_c3_fuse.py 2>&1 | head -3
done; } > gpurun_out/r2_split_policy.txt 2>&1

# latency configs against the cluster split-K width (CTAs per cluster at most: 8 default, 4, 2; red.add as reference)
mkdir -p gpurun_out
{ for v in default cs4 cs2 nocs default; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib python profiles/r2_c3_fuse.py 2>&1 | head -3
done; } > gpurun_out/r2_csplit_max.txt 2>&1

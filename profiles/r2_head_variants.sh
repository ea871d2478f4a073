# A/B of whole-head ring configurations (variants/lib_*.so), 512-instance launches
mkdir -p gpurun_out
for v in headold h1 h2 h4 h5 default; do
  if [ $v = default ]; then lib=paper_2009_07482_b200/libhetsim.so; else lib=variants/lib_$v.so; fi
  echo "== $v"; HETSIM_LIB=$lib timeout 300 python profiles/head_probe.py 512 2>&1 | tail -1
done > gpurun_out/r2_head_variants.txt 2>&1

mkdir -p gpurun_out
{ echo "== default (RZ off)"; python profiles/r2_c3_fuse.py; echo "== RZ (32-column X tiles)"; HETSIM_LIB=variants/lib_rz.so python profiles/r2_c3_fuse.py;
  echo "== head probe"; for v in default rz; do lib=paper_2009_07482_b200/libhetsim.so; [ $v = rz ] && lib=variants/lib_rz.so; HETSIM_LIB=$lib python profiles/head_probe.py 1 64 2>&1 | tail -2; done; } > gpurun_out/r2_rz_latency.txt 2>&1

mkdir -p gpurun_out
{ echo "== cluster split-K"; python profiles/r2_c3_fuse.py; echo "== red.add split-K"; HETSIM_LIB=variants/lib_nocs.so python profiles/r2_c3_fuse.py; echo "== cluster split-K again"; python profiles/r2_c3_fuse.py; } > gpurun_out/r2_c3_fuse.txt 2>&1

# cluster split-K with the bulk-copy push reduction: parity, determinism, timeline, latency configs
mkdir -p gpurun_out
{ timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_guards.py -q -x 2>&1 | tail -2
timeout 300 python profiles/determinism_probe.py
for i in 1 2; do HETSIM_LIB=variants/lib_gemmtl.so timeout 120 python profiles/gemm_timeline.py 256 256 256 0; HETSIM_LIB=variants/lib_gemmtl.so timeout 120 python profiles/gemm_timeline.py 128 512 2048 0; done
timeout 300 python profiles/r2_c3_fuse.py; timeout 300 python profiles/r2_c3_fuse.py; } > gpurun_out/r2_csplit_push.txt 2>&1

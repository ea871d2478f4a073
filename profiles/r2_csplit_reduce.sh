mkdir -p gpurun_out
{ for i in 1 2; do HETSIM_LIB=variants/lib_gemmtl.so python profiles/gemm_timeline.py 256 256 256 0; HETSIM_LIB=variants/lib_gemmtl.so python profiles/gemm_timeline.py 128 512 2048 0; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm_parity or split_k or head_fused_matches_grouped" 2>&1 | tail -2
python profiles/determinism_probe.py
python profiles/r2_c3_fuse.py; python profiles/r2_c3_fuse.py; } > gpurun_out/r2_csplit_reduce.txt 2>&1

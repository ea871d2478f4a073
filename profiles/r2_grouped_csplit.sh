mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
python profiles/r2_c3_fuse.py
python profiles/head_probe.py 1 2 2>&1 | tail -2
} > gpurun_out/r2_grouped_csplit.txt 2>&1

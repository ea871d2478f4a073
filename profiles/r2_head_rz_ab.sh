mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "head" 2>&1 | tail -5
echo "== new"; timeout 300 python profiles/head_probe.py 64 512 2>&1 | tail -6
echo "== old"; HETSIM_LIB=variants/lib_headold.so timeout 300 python profiles/head_probe.py 64 512 2>&1 | tail -6
} > gpurun_out/p5_head_rz.txt 2>&1

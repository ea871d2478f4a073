# RZ split with 32-column X tiles (SW128): correctness (tests with the variant lib) + timing + timeline
mkdir -p gpurun_out
{
HETSIM_LIB=variants/lib_x32a.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "head" 2>&1 | tail -3
for v in x32a headold; do echo "== $v"; HETSIM_LIB=variants/lib_$v.so timeout 300 python profiles/head_probe.py 64 512 2>&1 | tail -2; done
echo "== timeline x32"; HETSIM_LIB=variants/lib_tlx32.so timeout 300 python profiles/head_timeline.py 512 2>&1 | tail -12
} > gpurun_out/r2_head_x32.txt 2>&1

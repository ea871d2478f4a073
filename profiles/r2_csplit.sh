# cluster split-K: kernel parity + engine tests on one GPU, then the latency-config makespans
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_guards.py -q -x 2>&1 | tail -4
timeout 900 python profiles/run_graph_probe.py 2>&1 | tail -4
} > gpurun_out/r2_csplit.txt 2>&1

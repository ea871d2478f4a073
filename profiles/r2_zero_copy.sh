mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_engine_guards.py tests/test_gpu_engine.py -q -x 2>&1 | tail -3
timeout 900 python profiles/run_graph_probe.py 2>&1 | tail -8
} > gpurun_out/r2_zero_copy.txt 2>&1

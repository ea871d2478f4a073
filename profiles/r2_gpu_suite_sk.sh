mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_gputests.log
HETSIM_LIB=variants/lib_sk8.so python profiles/run_graph_probe.py > gpurun_out/run_graph_probe_sk8.txt 2>&1

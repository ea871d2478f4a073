mkdir -p gpurun_out
python profiles/determinism_probe.py > gpurun_out/determinism3.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_gputests.log
python profiles/run_graph_probe.py > gpurun_out/run_graph_probe2.txt 2>&1

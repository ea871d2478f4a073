# round-2 closing run: GPU suite, smoke, default bench line
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2i_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_smoke.log
python bench.py > gpurun_out/r2i_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_bench.log

# round-2 final: GPU suite, smoke, default bench line, 2-rank harness check on one GPU
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2g_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_smoke.log
python bench.py > gpurun_out/r2g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_bench.log
HS_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-alt --no-makespans > gpurun_out/r2g_bench_2ranks.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_bench_2ranks.log

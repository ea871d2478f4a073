# round-2 final (clean default library): GPU suite, smoke, bench line; cluster vs atomic split-K latency
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2h_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_smoke.log
python bench.py > gpurun_out/r2h_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_bench.log
{ echo "== cluster split-K (default library)"; python profiles/r2_c3_fuse.py;
  echo "== red.add split-K (variants/lib_nocs.so)"; HETSIM_LIB=variants/lib_nocs.so python profiles/r2_c3_fuse.py;
  echo "== cluster split-K again"; python profiles/r2_c3_fuse.py; } > gpurun_out/r2_csplit_vs_redadd.txt 2>&1

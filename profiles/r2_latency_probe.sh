# single-instance GEMM latency: clock64 timeline of CTA 0 (variant lib), graph-replay launch cost, small GEMMs
mkdir -p gpurun_out
{
for d in 0 1; do
  HETSIM_LIB=variants/lib_gemmtl.so python profiles/gemm_timeline.py 256 256 256 $d
  HETSIM_LIB=variants/lib_gemmtl.so python profiles/gemm_timeline.py 128 512 2048 $d
done
python profiles/latency_micro.py
python profiles/small_gemm.py
} > gpurun_out/r2_latency_probe.txt 2>&1

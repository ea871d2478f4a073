# C5 A/B: whole-head RZ default vs the previous head (variants/lib_headold.so), interleaved;
# C1-C4 makespans with split-K thresholds (variants/lib_sk4.so, lib_sk8.so)
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "head" 2>&1 | tail -2
for rep in 1 2; do
for v in default headold; do
  if [ $v = default ]; then lib=paper_2009_07482_b200/libhetsim.so; else lib=variants/lib_$v.so; fi
  HETSIM_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --no-alt --no-makespans 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['parity']['pass'], [round(r['ms_per_launch']*1e3,1) for r in d['roofline_other_kernels']])"
done; done
for v in default sk4 sk8; do
  if [ $v = default ]; then lib=paper_2009_07482_b200/libhetsim.so; else lib=variants/lib_$v.so; fi
  echo "== makespans $v"; HETSIM_LIB=$lib timeout 600 python profiles/pdl_probe.py 2>&1 | tail -3
done
} > gpurun_out/r2_ab_c5_latency.txt 2>&1

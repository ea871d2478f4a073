# lo terms rounded to tf32 (variants/lib_lorna.so, HS_LO_RNA=1): the 13 low bits the MMA ignores are
# zero instead of random. Parity, sustained FFN1 power/clock, C5 A/B interleaved.
mkdir -p gpurun_out
{
HETSIM_LIB=variants/lib_lorna.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
for v in default lorna default lorna; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib python profiles/power_probe.py 3 2>&1 | tail -1
done
for rep in 1 2; do
for v in default lorna; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  HETSIM_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --no-alt --no-makespans 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['parity']['pass'], d['parity']['normwise_vs_oracle'], d['parity']['normwise_vs_f64'])"
done; done
} > gpurun_out/r2_lo_rna.txt 2>&1

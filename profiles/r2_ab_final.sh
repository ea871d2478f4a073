# clean A/B after the variant-build fix: C5 default (head RZ off) vs variants/lib_rz.so, interleaved;
# FFN1 power / clock: default vs no-conversion vs MMA-only variants
mkdir -p gpurun_out
{
for rep in 1 2; do
for v in default rz; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  HETSIM_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --no-alt --no-makespans 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['parity']['pass'], [round(r['ms_per_launch']*1e3,1) for r in d['roofline_other_kernels']], round(d['roofline']['achieved'],1))"
done; done
nvidia-smi -q -d POWER | grep -iE "current power limit" | head -1
for v in default noconv mmaonly; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib python profiles/power_probe.py 3 2>&1 | tail -2
done
} > gpurun_out/r2_ab_final.txt 2>&1

mkdir -p gpurun_out
{
nvidia-smi -q -d POWER | grep -iE "limit|draw" | head -12
for v in default noconv mmaonly; do
  lib=paper_2009_07482_b200/libhetsim.so; [ $v != default ] && lib=variants/lib_$v.so
  echo "== $v"; HETSIM_LIB=$lib python profiles/power_probe.py 3 2>&1 | tail -2
done
} > gpurun_out/r2_power.txt 2>&1

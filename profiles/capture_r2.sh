#!/bin/bash
# Round-2 profiling recipe, run under gpurun from the repo root:
#  1. launch list of a short C5 bench run (batch 512), cold-cache and serialised
#  2. ncu --set full of the whole-head kernel (HS_OP_HEAD, head_kernel) at batch 512
#  3. ncu --set full of FFN1 (CTA-pair GEMM, tf32x3) at batch 512
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 1 --warmup 1 --instances 1024 --no-alt --no-e2e --no-cpu-baseline --no-makespans \
    > gpurun_out/r2_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^head_kernel" -s 3 -c 1 \
    -o gpurun_out/r2_head512 -f python profiles/head_probe.py 512 > gpurun_out/r2_head512.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -s 3 -c 1 \
    -o gpurun_out/r2_ffn1_512 -f python profiles/ffn1_probe.py tf32x3 512 1 > gpurun_out/r2_ffn1.log 2>&1
for r in r2_head512 r2_ffn1_512; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
cuobjdump -sass build/cuda/head_fused.o | grep -oE "UTCHMMA[.A-Z0-9]*|UTCQMMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG|LDTM[.A-Z0-9]*|STTM[.A-Z0-9]*|HMMA[.A-Z0-9]*" \
    | sort | uniq -c > gpurun_out/r2_head_sass_mnemonics.txt
ls -la gpurun_out

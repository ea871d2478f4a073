#!/bin/bash
# Profiling recipe for one round (run under gpurun from the repo root):
#  1. launch list of a short C5 bench run (cold-cache, serialised: compare shares)
#  2. ncu --set full of the dominant kernel (FFN1 on the CTA-pair GEMM) in both math modes
#  3. ncu --set full of the fused attention head
# Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
set -x
R=${1:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 1 --warmup 1 --instances 512 --no-alt --no-e2e --no-cpu-baseline \
    > gpurun_out/${R}_launches_bench.log 2>&1
for m in tf32x3 bf16x3; do
  ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -s 3 -c 1 \
      -o gpurun_out/${R}_ffn1_${m} -f python profiles/ffn1_probe.py $m 256 1 > gpurun_out/${R}_ffn1_${m}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:attn_head_kernel -s 3 -c 1 \
    -o gpurun_out/${R}_attn -f python profiles/attn_probe.py 256 > gpurun_out/${R}_attn.log 2>&1
ls -la gpurun_out

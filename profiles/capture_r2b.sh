#!/bin/bash
# Round-2 second-session captures (run under gpurun from the repo root):
#  1. ncu --set full of one cluster split-K launch: FFN2 at one instance (128x512x2048,
#     resident weight; 8 output tiles x 8 K-splits = 64 CTAs in clusters of 8)
#  2. launch list of a short C5 bench run with the final library (batch 512)
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 3 -c 1 \
    -o gpurun_out/r2b_csplit_ffn2 -f python profiles/one_gemm.py 128 512 2048 1 > gpurun_out/r2b_csplit.log 2>&1
ncu -i gpurun_out/r2b_csplit_ffn2.ncu-rep --page raw --csv > gpurun_out/r2b_csplit_ffn2_raw.csv 2>/dev/null
ncu -i gpurun_out/r2b_csplit_ffn2.ncu-rep --page details --csv > gpurun_out/r2b_csplit_ffn2_details.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
    python bench.py --steps 1 --warmup 1 --instances 1024 --no-alt --no-e2e --no-cpu-baseline --no-makespans \
    > gpurun_out/r2b_launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/r2b_launches.csv > gpurun_out/r2b_launches.txt

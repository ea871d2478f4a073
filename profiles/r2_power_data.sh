# is the FFN1 GEMM's sustained speed data-dependent (tensor-core power)? same kernel, operands random / zeros / ones
mkdir -p gpurun_out
for f in random zeros ones random; do python profiles/power_probe.py 3 $f 2>&1 | tail -1; done > gpurun_out/r2_power_data.txt 2>&1

mkdir -p gpurun_out
for d in 1 2 3 9; do
  python bench.py --devices $d --no-cpu-baseline --no-e2e --no-alt --no-makespans 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('devices', $d, d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['pass'])"
done > gpurun_out/probe1_devices.txt 2>&1
python profiles/latency_trace.py C1 > gpurun_out/probe1_trace_C1.txt 2>&1
python profiles/latency_trace.py C3 > gpurun_out/probe1_trace_C3.txt 2>&1

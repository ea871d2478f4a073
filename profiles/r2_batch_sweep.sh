# C5 device-resident throughput against the batch per launch and the slot count
mkdir -p gpurun_out
for cfg in "512 3" "1024 2" "1024 3" "768 3" "2048 2"; do
  set -- $cfg
  python bench.py --batch $1 --slots $2 --no-cpu-baseline --no-e2e --no-alt --no-makespans 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch', $1, 'slots', $2, round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['parity']['pass'], d['device_bytes']//2**20, 'MiB')"
done > gpurun_out/r2_batch_sweep.txt 2>&1

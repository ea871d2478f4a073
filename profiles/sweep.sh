#!/bin/bash
# Parameter sweep of the C5 bench (device-resident arm only): batch x logical devices x queues.
for cfg in "128 1 3" "128 9 3" "256 9 3" "256 1 3" "64 9 3"; do
  set -- $cfg
  v=$(timeout 200 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --batch $1 --devices $2 --queues $3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])" 2>/dev/null)
  echo "batch=$1 devices=$2 queues=$3 -> $v"
done

#!/bin/bash
# Parameter sweep of the C5 bench (device-resident arm only): batch x logical devices x queues [x math].
# usage: bash profiles/sweep.sh ["batch devices queues math" ...]
CFGS=("$@")
[ ${#CFGS[@]} -eq 0 ] && CFGS=("256 1 3 tf32x3" "296 1 3 tf32x3" "384 1 3 tf32x3" "512 1 3 tf32x3" "256 9 3 tf32x3" "512 9 3 tf32x3")
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  v=$(timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alt --batch $1 --devices $2 --queues $3 --math ${4:-tf32x3} 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])" 2>/dev/null)
  echo "batch=$1 devices=$2 queues=$3 math=${4:-tf32x3} -> $v"
done

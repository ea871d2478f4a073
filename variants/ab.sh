#!/bin/bash
# A/B a probe script across library variants inside one GPU session:
#   variants/ab.sh [probe.py args...]   (default: profiles/gemm_micro.py)
P=${1:-profiles/gemm_micro.py}; shift
for v in variants/lib_*.so; do echo "== $v"; HETSIM_LIB=$v timeout 120 python $P "$@" 2>&1 | tail -12; done

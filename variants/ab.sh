#!/bin/bash
# A/B the GEMM microbenchmark across library variants inside one GPU session.
for v in variants/lib_*.so; do echo "== $v"; HETSIM_LIB=$v timeout 120 python profiles/gemm_micro.py 2>&1 | grep -E "grouped|K=  512 batch= 148|2048 K=  512 batch= 128|512 K= 2048 batch= 128"; done

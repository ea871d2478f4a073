#!/bin/bash
# Build GEMM variants: variants/build.sh name "NVEXTRA flags"
set -e
touch paper_2009_07482_b200/csrc/cuda/*.cu
make -j8 NVEXTRA="$2" >/dev/null 2>&1 || { echo "build $1 failed"; make NVEXTRA="$2" 2>&1 | grep error | head; exit 1; }
cp paper_2009_07482_b200/libhetsim.so variants/lib_$1.so

#!/bin/bash
# Build a library variant in its own object directory, leaving the default build
# (build/, paper_2009_07482_b200/libhetsim.so) untouched:
#   variants/build.sh name "NVEXTRA flags"   -> variants/lib_name.so
set -e
make -j8 BUILD=build_var_$1 LIB=variants/lib_$1.so NVEXTRA="$2" variants/lib_$1.so >/dev/null 2>&1 || {
  echo "build $1 failed"; make BUILD=build_var_$1 LIB=variants/lib_$1.so NVEXTRA="$2" variants/lib_$1.so 2>&1 | grep error | head; exit 1; }

#!/bin/bash
# Build a tuning variant of the library: tools/build_variant.sh NAME -DMACRO=V ...
# -> paper_1805_04154_b200/librunsort_b200_NAME.so (select with RS_LIB=...)
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math \
  -Xcompiler -fPIC -shared "$@" -o paper_1805_04154_b200/librunsort_b200_$name.so paper_1805_04154_b200/csrc/runsort_b200.cu

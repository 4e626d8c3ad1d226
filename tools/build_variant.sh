#!/bin/bash
# Build a variant of libspdp.so with extra compile definitions (tuning experiments).
# usage: bash tools/build_variant.sh OUT.so -DKNOB=value ...   (then SPDP_LIB=OUT.so python bench.py ...)
out=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  paper_1510_06549_b200/csrc/spdp.cu -o "$out" -ldl -lpthread

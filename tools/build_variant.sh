#!/bin/bash
# Build an alternative library for A/B timing: build/NAME.so with extra -D flags.
#   bash tools/build_variant.sh NAME "-DKNOB=VALUE ..."
mkdir -p build
cd "$(dirname "$0")/../paper_1704_08579_b200/csrc" && \
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared \
  -gencode arch=compute_100a,code=sm_100a $2 -o ../../build/$1.so vexsort_b200.cu

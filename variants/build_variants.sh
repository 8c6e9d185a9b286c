#!/bin/bash
# experiment builds of the library with LCRW_EPI_MODE variants (not shipped)
set -e
cd "$(dirname "$0")/.."
for mode in ${MODES:-1 2 3}; do
  mkdir -p variants/m$mode
  for f in abi prep phase1 phase2 topk pipeline emd table; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DLCRW_EPI_MODE=$mode -c paper_1711_07227_b200/csrc/$f.cu -o variants/m$mode/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/m$mode/liblcrwmd.so variants/m$mode/*.o
done

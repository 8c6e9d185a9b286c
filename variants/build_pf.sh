#!/bin/bash
# prefetch-distance variants -> variants/pf$D/liblcrwmd.so
set -e
cd "$(dirname "$0")/.."
for D in ${PFS:-0 2 8}; do
  mkdir -p variants/pf$D
  for f in abi prep phase1 phase2 topk pipeline emd table; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DLCRW_P1_PREFETCH=$D ${EXTRA} -c paper_1711_07227_b200/csrc/$f.cu -o variants/pf$D/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/pf$D/liblcrwmd.so variants/pf$D/*.o
done

#!/bin/bash
# instrumented build (clock64 counters per role) -> variants/stats/liblcrwmd.so
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/stats
for f in abi prep phase1 phase2 topk pipeline emd table; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DLCRW_P1_STATS ${EXTRA} -c paper_1711_07227_b200/csrc/$f.cu -o variants/stats/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/stats/liblcrwmd.so variants/stats/*.o

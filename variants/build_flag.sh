#!/bin/bash
# experiment build of the library with one extra -D flag: NAME=dir FLAG=-DX=Y variants/build_flag.sh
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/$NAME
for f in $(python -c 'from paper_1711_07227_b200._build import SOURCES; print(" ".join(s[:-3] for s in SOURCES))'); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude $FLAG -c paper_1711_07227_b200/csrc/$f.cu -o variants/$NAME/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$NAME/liblcrwmd.so variants/$NAME/*.o

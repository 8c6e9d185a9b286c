#!/bin/bash
# experiment builds of csrc/refine.cu (not shipped): VARIANTS="name:-DFLAG=VALUE ..." variants/build_refine_variants.sh
set -e
cd "$(dirname "$0")/.."
for spec in $VARIANTS; do
  name=${spec%%:*}; flags=${spec#*:}; flags=${flags//,/ }
  mkdir -p variants/r_$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $flags \
       -Xptxas -v -c paper_1711_07227_b200/csrc/refine.cu -o variants/r_$name/refine.o 2> variants/r_$name/ptxas.log
  objs=$(ls paper_1711_07227_b200/build/*.o | grep -v '/refine.o$')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/r_$name/liblcrwmd.so $objs variants/r_$name/refine.o
  echo "$name: $(grep -A3 refine_kernel variants/r_$name/ptxas.log | grep -o 'Used [0-9]* registers') $(grep -A3 refine_kernel variants/r_$name/ptxas.log | grep -o '[0-9]* bytes spill stores')"
done

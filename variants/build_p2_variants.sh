#!/bin/bash
# experiment builds of csrc/phase2.cu (A/B of spmm / reverse_panels shapes; not shipped):
#   VARIANTS="name:-DFLAG=VALUE ..." variants/build_p2_variants.sh  (compile-time knobs of phase2.cu)
set -e
cd "$(dirname "$0")/.."
for spec in $VARIANTS; do
  name=${spec%%:*}
  flags=${spec#*:}
  flags=${flags//,/ }
  mkdir -p variants/s_$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $flags \
       -Xptxas -v -c paper_1711_07227_b200/csrc/phase2.cu -o variants/s_$name/phase2.o 2> variants/s_$name/ptxas.log &
done
wait
for spec in $VARIANTS; do
  name=${spec%%:*}
  objs=$(ls paper_1711_07227_b200/build/*.o | grep -v '/phase2.o$')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/s_$name/liblcrwmd.so $objs variants/s_$name/phase2.o
  echo "$name: $(grep -A2 spmm_kernel variants/s_$name/ptxas.log | grep -o 'Used [0-9]* registers')"
done

#!/bin/bash
# experiment builds of csrc/table.cu (A/B of table_min shapes; not shipped):
#   VARIANTS="m4:-DLCRW_TBL_MINB=4 m6:-DLCRW_TBL_MINB=6 ..." variants/build_table_variants.sh
# (the round-2 A/B knobs that lost were removed from table.cu; profiles/r02_summary.md lists them)
# each variant links the shipped objects of paper_1711_07227_b200/build with its own table.o
set -e
cd "$(dirname "$0")/.."
for spec in $VARIANTS; do
  name=${spec%%:*}
  flags=${spec#*:}
  flags=${flags//,/ }
  mkdir -p variants/t_$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $flags \
       -Xptxas -v -c paper_1711_07227_b200/csrc/table.cu -o variants/t_$name/table.o 2> variants/t_$name/ptxas.log &
done
wait
for spec in $VARIANTS; do
  name=${spec%%:*}
  objs=$(ls paper_1711_07227_b200/build/*.o | grep -v '/table.o$')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/t_$name/liblcrwmd.so $objs variants/t_$name/table.o
  echo "$name: $(grep -A2 table_min variants/t_$name/ptxas.log | grep -o 'Used [0-9]* registers')"
done

#!/bin/bash
# Build an experiment variant of the library: tools/variant.sh NAME "-DMACRO=..." [unit ...]
# recompiles the named translation units (default inst_u32.cu, the headline engine) with the
# extra flags into paper_2407_14801_b200/build_NAME/ and links them with the default build's
# other objects into paper_2407_14801_b200/libsq_NAME.so (use with SQ_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; shift 2
units=${@:-inst_u32.cu}
P=paper_2407_14801_b200
mkdir -p $P/build_$name
objs=""
for o in $P/build/*.o; do
  b=$(basename $o .o)
  if [[ " $units " == *" $b.cu "* ]]; then
    nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC $flags -c -o $P/build_$name/$b.o $P/csrc/$b.cu &
    objs="$objs $P/build_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libsq_$name.so $objs
echo built $P/libsq_$name.so

#!/bin/bash
# Builds library variants with one source recompiled under -D overrides,
# linked with the tree's other objects, into altlib/<name>/librunq_b200.so
# usage: bash tools/lib_variants.sh <source.cu> name1 "-DX=1 ..." name2 "..."
set -u
src=$1; shift
obj=$(basename $src .cu).o
(cd paper_2506_10092_b200/csrc && make -s -j8)
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills"
names=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p altlib/$name/obj
  $NV $flags -c paper_2506_10092_b200/csrc/$src -o altlib/$name/obj/$obj &
  names+=($name)
done
wait
objs=$(ls build/obj/*.o | grep -v "/$obj")
for name in "${names[@]}"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o altlib/$name/librunq_b200.so $objs altlib/$name/obj/$obj -ldl -Xlinker --exclude-libs,ALL && echo built $name
done

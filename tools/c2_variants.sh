#!/bin/bash
# Builds C2 TMA-kernel shape variants (k_fused.cu recompiled with -D overrides,
# linked with the tree's other objects) into altlib/<name>/librunq_b200.so
# usage: bash tools/c2_variants.sh name1 "-DRQ_C2_TI=2 ..." name2 "..."
set -eu
cd paper_2506_10092_b200/csrc && make -s -j8 && cd ../..
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=altlib/$name; mkdir -p $d/obj
  $NV $flags -c paper_2506_10092_b200/csrc/k_fused.cu -o $d/obj/k_fused.o &
done
wait
for d in altlib/*/; do
  [ -f $d/obj/k_fused.o ] || continue
  objs=$(ls build/obj/*.o | grep -v k_fused.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/librunq_b200.so $objs $d/obj/k_fused.o -ldl -Xlinker --exclude-libs,ALL
  echo built $d
done

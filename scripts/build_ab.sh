#!/bin/bash
# A/B builds of k_wave2's level-0 ring (PTB_WAVE2_RING variants, see propagate.cu):
#   paratime_b200/_ab/libparatime_b200_ring<V>.so for each V given (default 1 2 3); load one with
#   PTB_LIB=... (measurements only; the default build is the product)
set -e
cd "$(dirname "$0")/.."
mkdir -p paratime_b200/_ab
B=paratime_b200/_build
NCCL_INC=$(python -c "import paratime_b200.build as b; print(b._nccl_include())")
objs=$(ls $B/*.o | grep -v propagate_cu.o | tr "\n" " ")
for V in ${@:-1 2 3}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -Iinclude \
    -Iparatime_b200/csrc -I"$NCCL_INC" --expt-relaxed-constexpr -DPTB_WAVE2_RING=$V \
    -x cu -c paratime_b200/csrc/propagate.cu -o paratime_b200/_ab/propagate_ring$V.o &
done
wait
for V in ${@:-1 2 3}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paratime_b200/_ab/libparatime_b200_ring$V.so \
    $objs paratime_b200/_ab/propagate_ring$V.o -lcudart -ldl
  echo built paratime_b200/_ab/libparatime_b200_ring$V.so
done

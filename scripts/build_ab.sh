#!/bin/bash
# A/B build: the library with k_wave2's round-1 per-thread cp.async ring (PTB_WAVE2_CPASYNC=1)
# -> paratime_b200/_ab/libparatime_b200_cpasync.so (load with PTB_LIB=...; measurements only)
set -e
cd "$(dirname "$0")/.."
mkdir -p paratime_b200/_ab
B=paratime_b200/_build
NCCL_INC=$(python -c "import paratime_b200.build as b; print(b._nccl_include())")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -Iinclude \
  -Iparatime_b200/csrc -I"$NCCL_INC" --expt-relaxed-constexpr -DPTB_WAVE2_CPASYNC=1 \
  -x cu -c paratime_b200/csrc/propagate.cu -o paratime_b200/_ab/propagate_cpasync.o
objs=$(ls $B/*.o | grep -v propagate_cu.o | tr "\n" " ")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paratime_b200/_ab/libparatime_b200_cpasync.so \
  $objs paratime_b200/_ab/propagate_cpasync.o -lcudart -ldl
echo built paratime_b200/_ab/libparatime_b200_cpasync.so

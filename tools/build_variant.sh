#!/bin/bash
# Build a variant of libgamblets_b200.so with extra nvcc defines for A/B
# timing (load it with GB_LIB=<path>).  Usage: tools/build_variant.sh name -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
objs=""
for s in gb_box gb_patch gb_products gb_krylov gb_dense gb_diag gb_3d gb_capi; do
  nvcc $F "$@" -c paper_1503_03467_b200/csrc/$s.cu -o $out/$s.o &
  objs="$objs $out/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs -o $out/libgamblets_b200.so \
  -Xlinker -rpath=/usr/local/cuda/lib64
echo built $out/libgamblets_b200.so

#!/bin/bash
# Builds libposlo_gpu.so with extra -D flags as variant_<name>.so at the repo
# root (for the tools/gpu_ab_*.sh A/B runs): tools/build_variant.sh NAME "-DX=1 -DY=2"
set -e
cd "$(dirname "$0")/../paper_2506_08781_b200/csrc"
NAME=$1; shift
FLAGS="$*"
OUT=/tmp/poslo_variant_$NAME
mkdir -p $OUT
objs=""
for f in capi.cu multi.cu verify_kernels.cu hash_s1.cu hash_s2.cu hash_var.cu group_kernels.cu log_scan.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $FLAGS -c $f -o $OUT/${f%.cu}.o &
  objs="$objs $OUT/${f%.cu}.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../variant_$NAME.so $objs
echo "built variant_$NAME.so ($FLAGS)"

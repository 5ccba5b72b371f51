#!/bin/bash
# Build an alternative libpd_b200.so with extra nvcc defines, for A/B runs (load it with PD_LIB=...).
#   tools/build_variant.sh build/alt -DPD_MBAR_SUSPEND=0
set -e
out=$1; shift
mkdir -p $out/obj
cd "$(dirname "$0")/.."
for f in gemm kernels layers attention attention_tc transformer runtime; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include "$@" \
    -c paper_1806_03377_b200/csrc/$f.cu -o $out/obj/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpd_b200.so $out/obj/*.o
echo "built $out/libpd_b200.so"

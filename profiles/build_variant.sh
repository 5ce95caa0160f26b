#!/bin/bash
# A/B build of libqsb200.so with extra nvcc defines into var/NAME/ (travels with gpurun;
# select it with QS_LIB=var/NAME/libqsb200.so).   usage: profiles/build_variant.sh NAME -DQS_I4_KCH1=64 ...
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/var/$NAME; mkdir -p $OUT
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $ROOT/include $*"
for s in qs_attn qs_gemm qs_quant qs_ops qs_capi; do
  nvcc $F -c $ROOT/paper_2502_10424_b200/csrc/$s.cu -o $OUT/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libqsb200.so $OUT/*.o -lcudart
rm -f $OUT/*.o
echo $OUT/libqsb200.so

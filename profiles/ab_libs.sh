#!/bin/bash
# A/B of libqsb200.so builds (var/NAME/libqsb200.so from profiles/build_variant.sh; "" = in-tree)
# on the attention and GEMV microbenchmarks.   usage (under gpurun): bash profiles/ab_libs.sh OUT "" var/a var/b
OUT=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  lib=${L:+$L/libqsb200.so}
  echo "== lib=${lib:-in-tree}" >> gpurun_out/$OUT
  for ctx in 131072 32768; do
    QS_LIB=$lib timeout 300 python profiles/attn_micro.py --context $ctx --T 1,5,9 --graph 1 >> gpurun_out/$OUT 2>&1
  done
  QS_LIB=$lib timeout 300 python profiles/gemv_micro.py --modes f16,int4 --groups 32 >> gpurun_out/$OUT 2>&1
done

#!/bin/bash
# End-to-end A/B of libqsb200.so builds on the decode cycle (interleaved repetitions, one box).
#   usage (under gpurun): bash profiles/ab_bench.sh OUT LIBDIR|- ...    (- = in-tree build)
OUT=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
  for L in "$@"; do
    lib=""; [ "$L" != "-" ] && lib=$L/libqsb200.so
    echo "== lib=${lib:-in-tree} rep=$r" >> gpurun_out/$OUT
    QS_LIB=$lib QS_BENCH_NO_KERNELS=1 python bench.py --modes ${AB_MODES:-both,fp16_ar} --steps 32 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print({k:(round(v.get('tok_s'),2), v.get('acceptance'), round(v.get('ms_per_step'),3)) for k,v in d['modes'].items()}, d['clocks'])" >> gpurun_out/$OUT
  done
done

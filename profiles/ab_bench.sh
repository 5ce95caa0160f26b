for r in 1 2; do
for L in var/old_i4 ""; do
  echo "== lib=${L:-in-tree} rep=$r" >> gpurun_out/ab_bench.txt
  QS_LIB=${L:+$L/libqsb200.so} QS_BENCH_NO_KERNELS=1 python bench.py --modes both,fp16_ar --steps 32 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print({k:(round(v.get('tok_s'),2), v.get('acceptance'), round(v.get('ms_per_step'),3)) for k,v in d['modes'].items()}, d['clocks'])" >> gpurun_out/ab_bench.txt
done; done

#!/bin/bash
# ncu --set full captures of the hot kernels as launched by `bench.py --profile-kernels`
# (draft attention = 4th attn launch, verify = 27th, fp16-cache = 50th; then the f16 and
# INT4 GEMVs).  Summaries land in gpurun_out/TAG_summary.txt; only the draft report is kept.
TAG=${1:-r01}; SET=${2:-full}; KEEP=${3:-attn_draft}
mkdir -p gpurun_out
for spec in "attn_kernel 3 attn_draft" "attn_kernel 26 attn_verify" "attn_kernel 49 attn_fp16" "linear_f16p_kernel 3 gemv_f16" "linear_i4_kernel 3 gemv_int4"; do
  set -- $spec
  QS_BENCH_ISOLATED=1 timeout 900 ncu --set $SET --import-source on --clock-control none -k regex:$1 -s $2 -c 1 \
      -o /tmp/${TAG}_$3 python bench.py --profile-kernels > /tmp/${TAG}_$3.log 2>&1
  python profiles/summarize_ncu.py /tmp/${TAG}_$3.ncu-rep >> gpurun_out/${TAG}_summary.txt
done
cp /tmp/${TAG}_${KEEP}.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out

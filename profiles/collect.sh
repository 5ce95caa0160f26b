#!/bin/bash
# One GPU-box pass that refreshes the committed evidence for a round (run under gpurun):
#   1. ncu launch list of steady-state speculative cycles (our kernels only; cold-cache serialised
#      times: compare SHARES)                                    -> gpurun_out/${TAG}_launches.csv
#   2. ncu --set full summaries of the hot kernels               -> gpurun_out/${TAG}_summary.txt
#   3. ncu DRAM bytes of the draft-attention launch, tied to this build's md5 -> profiles/traffic.json
#   4. the attention context / gamma sweep + K1 flush            -> gpurun_out/${TAG}_sweep.txt
# Usage: bash profiles/collect.sh r02
TAG=${1:-r02}
mkdir -p gpurun_out
QS_BENCH_NO_KERNELS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:attn_kernel|linear_|prep_act|embed_kernel|argmax|accept|add_int|kv_quant|kv_flush|fp_rotate' \
    -s 400 -c 1400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --modes both > /tmp/${TAG}_ll.log 2>&1
python profiles/launch_shares.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_shares.txt 2>&1
timeout 2400 bash profiles/profile_kernels.sh ${TAG} full attn_draft
timeout 1200 bash profiles/collect_traffic.sh
timeout 900 python profiles/sweep.py > gpurun_out/${TAG}_sweep.txt 2>&1

#!/bin/bash
# compute-sanitizer over the kernel-level GPU parity tests (attention, linear, flush, ops) of the
# current build.   usage (under gpurun): bash profiles/sanitize.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
SEL="attention or linear or flush or quant or accept or argmax or embed"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > gpurun_out/sanitizer_${tool}_${TAG}.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_${tool}_${TAG}.txt
  tail -3 gpurun_out/sanitizer_${tool}_${TAG}.txt
done

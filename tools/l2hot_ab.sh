#!/bin/bash
# L2 hot-row window A/B through the bench (N=1), interleaved repeats.
set -u
mkdir -p gpurun_out
: > gpurun_out/l2hot.txt
for rep in 1 2 3; do
  for mb in ${L2HOT_SWEEP:-0 8 16}; do
    TIERSHARD_L2_HOT_MB=$mb timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-routing > gpurun_out/ab.json 2>&1
    tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('mb=$mb', d['value'], d['e2e']['value'])" >> gpurun_out/l2hot.txt
  done
done
cat gpurun_out/l2hot.txt

#!/bin/bash
# L2 persisting window over the hot rows, A/B at N=1 (one GPU).
set -u
mkdir -p gpurun_out
for mb in 0 16 32 64; do
  echo "== L2_HOT_MB=$mb"
  TIERSHARD_L2_HOT_MB=$mb timeout 600 python tools/h2d_probe.py 2>&1 | grep -E "ms/step"
done

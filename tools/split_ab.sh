#!/bin/bash
# SM-partition A/B at N=1 (run under gpurun on one GPU): parity tests with a
# split, then the N=1 step for each K.
set -u
mkdir -p gpurun_out
TIERSHARD_SM_SPLIT=16 timeout 600 python -m pytest tests/test_gpu_table.py -q -x > gpurun_out/split_pytest.log 2>&1; tail -1 gpurun_out/split_pytest.log
B="python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-routing"
: > gpurun_out/split_ab.txt
for v in "$@"; do
  env $v timeout 600 $B > gpurun_out/ab.json 2> gpurun_out/ab.err
  tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])" >> gpurun_out/split_ab.txt 2>&1
done
cat gpurun_out/split_ab.txt

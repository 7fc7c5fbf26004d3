#!/bin/bash
# Cross-step dedup (lookahead) A/B at N=1 (run under gpurun on one GPU).
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_table.py tests/test_plan_import.py -q -x > gpurun_out/la.log 2>&1; tail -1 gpurun_out/la.log
B="python bench.py --no-cpu-baseline --no-routing"
timeout 600 $B > gpurun_out/la_on.json 2> gpurun_out/la_on.err
TIERSHARD_LOOKAHEAD=0 timeout 600 $B > gpurun_out/la_off.json 2>&1
TIERSHARD_LA_GATHER_BLOCKS=5 timeout 600 $B > gpurun_out/la_on5.json 2>&1
TIERSHARD_LA_GATHER_BLOCKS=8 timeout 600 $B > gpurun_out/la_on8.json 2>&1
for f in la_on la_off la_on5 la_on8; do
  tail -1 gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$f', d['value'], d['e2e']['value'], d['e2e'].get('step_trace_ms'))"
done

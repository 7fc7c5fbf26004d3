#!/bin/bash
# A/B the short-segment kernel variants on the default N=1 bench (under gpurun).
timeout 600 python -m pytest tests/test_gpu_table.py -q -x 2>&1 | tail -1
for v in "TIERSHARD_SEG=single" "TIERSHARD_SEG=pair TIERSHARD_SEG_G=16" "TIERSHARD_SEG=pair TIERSHARD_SEG_G=8"; do
  env $v timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])"
done

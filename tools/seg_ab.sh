#!/bin/bash
# A/B segment-phase schedules on the default N=1 bench (under gpurun):
# long segments concurrent with the short kernel or after it, and the
# gather's blocks per SM while the dedup sort runs beside it.
timeout 600 python -m pytest tests/test_gpu_table.py -q -x 2>&1 | tail -1
for v in "TIERSHARD_LONG_CONCURRENT=1" "TIERSHARD_LONG_CONCURRENT=0" \
         "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_GATHER_BLOCKS=6" "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_GATHER_BLOCKS=4" \
         "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_SHORT_MAX=64" "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_SHORT_MAX=16" \
         "TIERSHARD_LONG_CONCURRENT=1" "TIERSHARD_LONG_CONCURRENT=0"; do
  env $v timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'])"
done

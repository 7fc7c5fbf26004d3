#!/bin/bash
# N=1 A/B: the short-segment kernel's blocks per SM while the long path runs beside it.
for v in "TIERSHARD_SHORT_BLOCKS=8" "TIERSHARD_SHORT_BLOCKS=4" "TIERSHARD_SHORT_BLOCKS=3" "TIERSHARD_SHORT_BLOCKS=2" "TIERSHARD_SHORT_BLOCKS=8" "TIERSHARD_SHORT_BLOCKS=3"; do
  env $v timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'], d['step_trace_ms'] if 'step_trace_ms' in d else '')"
done

for v in "TIERSHARD_AUX_PRIORITY=low" "TIERSHARD_AUX_PRIORITY=high" "TIERSHARD_AUX_PRIORITY=high TIERSHARD_GATHER_BLOCKS=4" "TIERSHARD_AUX_PRIORITY=high TIERSHARD_GATHER_BLOCKS=6" "TIERSHARD_AUX_PRIORITY=low" "TIERSHARD_AUX_PRIORITY=high"; do
  env $v timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print('$v', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'], d['roofline']['frac'])"
done

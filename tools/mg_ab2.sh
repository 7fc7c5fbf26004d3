#!/bin/bash
# N=$NGPU A/B: aux (dedup) stream priority and the gather's blocks per SM.
N=${NGPU:-2}
for v in "TIERSHARD_AUX_PRIORITY=low" "TIERSHARD_AUX_PRIORITY=high" "TIERSHARD_AUX_PRIORITY=low TIERSHARD_GATHER_BLOCKS=6" \
         "TIERSHARD_AUX_PRIORITY=high TIERSHARD_GATHER_BLOCKS=6" "TIERSHARD_AUX_PRIORITY=low" "TIERSHARD_AUX_PRIORITY=high"; do
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads([l for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]);print('$v', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'])"
done

#!/bin/bash
# Multi-GPU parity tests, then an A/B of the segment schedule at N=$NGPU.
N=${NGPU:-2}
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_table.py -x -q 2>&1 | tail -1
for v in "TIERSHARD_LONG_CONCURRENT=1" "TIERSHARD_LONG_CONCURRENT=0" "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_SHORT_MAX=64" \
         "TIERSHARD_LONG_CONCURRENT=1 TIERSHARD_SHORT_MAX=32" "TIERSHARD_LONG_CONCURRENT=1" "TIERSHARD_LONG_CONCURRENT=0"; do
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads([l for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]);print('$v', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'])"
done

#!/bin/bash
# Sweep the U>1 schedule knobs with the 2-rank bench (run under gpurun --gpus 2).
for rep in concurrent serial; do
  for pull in 0 1; do
    TIERSHARD_REPLICA=$rep TIERSHARD_PULL_GRADS=$pull timeout 600 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node ${NGPU:-2} --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus ${NGPU:-2} \
      --steps 30 --warmup 5 --no-e2e > gpurun_out/sweep_${rep}_${pull}.json 2> gpurun_out/sweep_${rep}_${pull}.err
    python -c "
import json,sys;d=json.loads(open('gpurun_out/sweep_${rep}_${pull}.json').read().splitlines()[-1])
print('${rep} pull=${pull}', d['value'], d['ms_per_step'], [(r[0],r[1],round(r[3]-r[2],3)) for r in d['step_trace_ms']])"
  done
done

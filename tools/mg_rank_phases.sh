#!/bin/bash
# Per-rank phase means and one step's timeline on every rank (run under
# gpurun --gpus N): bench.py with TS_BENCH_DIAG=1.
set -u
N=${1:-4}
mkdir -p gpurun_out
TS_BENCH_DIAG=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29581 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline ${BENCH_EXTRA:-} \
  > gpurun_out/rank_phases_n$N.json 2> gpurun_out/rank_phases_n$N.err
tail -1 gpurun_out/rank_phases_n$N.json | python -c "
import json, sys
d = json.loads(sys.stdin.readline())
for r, ph in enumerate(d['phases_ms_all_ranks']):
    print('rank', r, ph)
for r, tr in enumerate(d['step_trace_ms_all_ranks']):
    print('rank', r, tr)
"

#!/bin/bash
# N-GPU A/B of the forward gather variant (run under gpurun --gpus N).
set -u
N=${1:-2}; shift
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29566 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
: > gpurun_out/mg_gather_ab.txt
for v in "$@"; do
  set -- $v
  TIERSHARD_GATHER=$1 TIERSHARD_GATHER_BLOCKS=$2 TIERSHARD_BULK_STAGES=$3 timeout 600 $R ${4:-} > gpurun_out/ab.json 2> gpurun_out/ab.err
  tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['nvlink']['frac'], d['roofline']['all_phases_ms_per_step'])" >> gpurun_out/mg_gather_ab.txt 2>&1
done
cat gpurun_out/mg_gather_ab.txt

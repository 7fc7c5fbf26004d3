#!/bin/bash
# N-GPU A/B over environment settings (run under gpurun --gpus N):
#   bash tools/mg_env_ab.sh N "ENV=a ENV2=b|label" ... [-- extra bench args]
set -u
N=$1; shift
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline ${BENCH_EXTRA:-}"
: > gpurun_out/mg_env_ab.txt
for v in "$@"; do
  envs=${v%%|*}; label=${v##*|}
  env $envs timeout 600 $R > gpurun_out/ab.json 2> gpurun_out/ab.err
  tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$label', d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['nvlink']['frac'], d['roofline']['all_phases_ms_per_step'])" >> gpurun_out/mg_env_ab.txt 2>&1
done
cat gpurun_out/mg_env_ab.txt

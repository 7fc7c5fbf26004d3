#!/bin/bash
# N=4 A/B of the gradient-push grid (run under gpurun --gpus 4): C2, 1 x 4
# and 2 x 2 virtual nodes, TIERSHARD_PUSH_BLOCKS = 1 / 2 / 4 per SM.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -x -k "2-2 or 2-4 or 2-1" > gpurun_out/mg_ab_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/mg_ab_pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline"
: > gpurun_out/mg_ab.txt
for vn in "" "--virtual-nodes"; do
  for pb in 1 2 4; do
    TIERSHARD_PUSH_BLOCKS=$pb timeout 600 $R $vn > gpurun_out/ab.json 2> gpurun_out/ab.err
    tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('vn=$vn push=$pb', d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['nvlink']['frac'], d['roofline']['all_phases_ms_per_step'])" >> gpurun_out/mg_ab.txt 2>&1
  done
done
cat gpurun_out/mg_ab.txt

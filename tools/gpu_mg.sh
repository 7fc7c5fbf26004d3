#!/bin/bash
# Multi-GPU pass (run under gpurun --gpus N): the multi-rank tests on real
# GPUs, then the N-GPU bench line (1 x N, 2-tier) and, at N = 4, 2 x 2
# virtual nodes (3-tier).  Outputs in gpurun_out/.
set -u
N=${1:-2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/mg_pytest_n$N.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/mg_pytest_n$N.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N"
timeout 900 $R > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench_rc=$?; tail -2 gpurun_out/bench_n$N.err
if [ "$N" = "4" ]; then
  timeout 900 $R --virtual-nodes > gpurun_out/bench_n4_vn.json 2> gpurun_out/bench_n4_vn.err; echo bench_vn_rc=$?
fi

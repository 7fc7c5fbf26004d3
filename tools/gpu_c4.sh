#!/bin/bash
# Full C4 on a 4-GPU lease (run under gpurun --gpus 4): 16 tables x 50M rows
# x D=128, L = 256/table, batch 4096/GPU, 2 x 2 virtual nodes, 3-tier,
# GPU-sampled batches.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
free -g > gpurun_out/c4_host_mem.txt 2>&1
timeout 3000 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 \
  bench.py --gpus 4 --tables 16 --rows 50000000 --seq-len 256 --virtual-nodes --sampler gpu --steps 10 --warmup 3 \
  > gpurun_out/bench_c4_n4.json 2> gpurun_out/bench_c4_n4.err; echo c4_rc=$?; tail -3 gpurun_out/bench_c4_n4.err

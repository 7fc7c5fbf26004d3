#!/bin/bash
# Round-end multi-GPU evidence (gpurun --gpus 4): full GPU test suite, then
# bench lines at N=2 (GPUs 0,1), N=4 (1x4) and N=4 (2x2 virtual nodes, 3-tier).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu4.log; tail -2 gpurun_out/pytest_gpu4.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 > gpurun_out/fin_n2.json 2> gpurun_out/fin_n2.err; echo n2=$?
timeout 600 $R --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 > gpurun_out/fin_n4.json 2> gpurun_out/fin_n4.err; echo n4=$?
timeout 600 $R --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --virtual-nodes > gpurun_out/fin_n4vn.json 2> gpurun_out/fin_n4vn.err; echo n4vn=$?
for f in fin_n2 fin_n4 fin_n4vn; do
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/$f.json') if l.startswith('{')][-1])
print('$f', d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), d['nvlink']['frac'], d['lookup_exchange'].get('samples_per_s'))
PY
done

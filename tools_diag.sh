mkdir -p gpurun_out
TS_BENCH_DIAG=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 30 --warmup 5 --virtual-nodes > gpurun_out/vn4.json 2> gpurun_out/vn4.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/vn4.json') if l.startswith('{')][-1])
print('N=4 2x2 3tier', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], 'e2e', d['e2e']['value'])
print(d['config']); print(d['nvlink']); print(d['a2a'])
print(d['roofline']['all_phases_ms_per_step'])
PY

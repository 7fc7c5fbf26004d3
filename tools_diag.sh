mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_table.py tests/test_gpu_multigpu.py -x -q -k "pipelined or host or single or two_steps" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log; tail -2 gpurun_out/t.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/d1.json 2> gpurun_out/d1.err
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/d$N.json 2> gpurun_out/d$N.err
done
for N in 1 2 4; do
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/d$N.json') if l.startswith('{')][-1])
e=d['e2e']
print('N=$N', d['value'], d['ms_per_step'], 'e2e', round(e['value']), 'per-call', round(e['per_call_value']), e['per_call_step_wall_ms'])
PY
done

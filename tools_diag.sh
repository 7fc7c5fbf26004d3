mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/diag_n1.json 2> gpurun_out/diag_n1.err
for N in 2 4; do
TS_BENCH_DIAG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/diag_n$N.json 2> gpurun_out/diag_n$N.err
done
for N in 1 2 4; do
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/diag_n$N.json') if l.startswith('{')][-1])
e=d.get('e2e') or {}
r=d['roofline']
print('N=$N', d['value'], d['ms_per_step'], 'e2e', e.get('value'), e.get('step_wall_ms'), 'diag', e.get('diag_torch_buffers_value'), e.get('diag_host_api_pinned_value'))
print('  ', r['all_phases_ms_per_step'])
PY
done

mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/diag_n1.json 2> gpurun_out/diag_n1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/diag_n2.json 2> gpurun_out/diag_n2.err
for n in 1 2; do
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/diag_n$n.json') if l.startswith('{')][-1])
e=d.get('e2e') or {}
r=d['roofline']
print('N=$n', d['value'], d['ms_per_step'], 'e2e', e.get('value'), e.get('step_wall_ms'), r['kernel'], r['achieved'], r['frac'])
print(r['all_phases_ms_per_step'])
for x in d.get('step_trace_ms', []): print('  ', x)
PY
done

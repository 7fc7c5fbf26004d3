mkdir -p gpurun_out
for N in 4; do
TS_BENCH_DIAG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/diag_n$N.json 2> gpurun_out/diag_n$N.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/diag_n$N.json') if l.startswith('{')][-1])
print('N=$N', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], 'e2e', d['e2e']['value'], d['clocks'])
for rk, tr in enumerate(d['step_trace_ms_all_ranks']):
    print('rank', rk, ' '.join(f"{n}:{s}:{a:.2f}-{b:.2f}" for n, s, a, b in tr))
PY
done

mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -x -q -k "p2p and not pull" > gpurun_out/mg.log 2>&1; echo rc=$? >> gpurun_out/mg.log; tail -2 gpurun_out/mg.log
for N in 2 4; do for rep in 1 2; do
TS_BENCH_DIAG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/d$N.json 2> gpurun_out/d$N.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/d$N.json') if l.startswith('{')][-1])
print('N=$N', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], 'e2e', round(d['e2e']['value']))
tr=d['step_trace_ms_all_ranks'][0]
print('   rank0', ' '.join(f"{n}:{s}:{a:.2f}-{b:.2f}" for n, s, a, b in tr))
PY
done; done

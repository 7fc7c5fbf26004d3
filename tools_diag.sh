mkdir -p gpurun_out
TIERSHARD_PUSH_ORDER=first timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q -k "p2p" > gpurun_out/mg_tests.log 2>&1; echo rc=$? >> gpurun_out/mg_tests.log
tail -2 gpurun_out/mg_tests.log
for po in overlap first; do
N=4
TIERSHARD_PUSH_ORDER=$po TS_BENCH_DIAG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > gpurun_out/diag_n4.json 2> gpurun_out/diag_n4.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/diag_n4.json') if l.startswith('{')][-1])
print('push_order=$po', d['value'], d['ms_per_step'])
for rk, tr in enumerate(d['step_trace_ms_all_ranks']):
    print('rank', rk, ' '.join(f"{n}:{s}:{a:.2f}-{b:.2f}" for n, s, a, b in tr))
PY
done

#!/bin/bash
# 2/4-rank checks: multi-GPU parity tests, then the bench at N=$NGPU (gpurun --gpus N).
N=${NGPU:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/mg_tests_n$N.log 2>&1; echo rc=$? >> gpurun_out/mg_tests_n$N.log
tail -3 gpurun_out/mg_tests_n$N.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/mg_bench_n$N.json 2> gpurun_out/mg_bench_n$N.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/mg_bench_n$N.json') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d.get('e2e',{}) and d['e2e']['value'])
print(d['roofline']['all_phases_ms_per_step'])
for r in d['step_trace_ms']: print('  ', r)
PY
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/mg_bench_n$N.json') if l.startswith('{')][-1])
e=d.get('e2e') or {}
print('e2e', e.get('value'), e.get('step_wall_ms'))
for r in e.get('step_trace_ms', []): print('  ', r)
PY

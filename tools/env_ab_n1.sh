#!/bin/bash
# N=1 A/B over environment settings through the bench (device value and
# e2e), interleaved repeats (run under gpurun):
#   REPS=2 bash tools/env_ab_n1.sh "ENV=a ENV2=b|label" ...
set -u
mkdir -p gpurun_out
: > gpurun_out/env_ab_n1.txt
for rep in $(seq 1 ${REPS:-2}); do
  for v in "$@"; do
    envs=${v%%|*}; label=${v##*|}
    env $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-routing > gpurun_out/ab.json 2> gpurun_out/ab.err
    tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('$label', d['value'], d['ms_per_step'], e['value'], e.get('pipelined_device_ms_per_step'))" >> gpurun_out/env_ab_n1.txt 2>&1
  done
done
cat gpurun_out/env_ab_n1.txt

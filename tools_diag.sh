mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not multigpu" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for r9 in 0 1; do for dif in 0 1; do
TIERSHARD_RADIX9=$r9 TIERSHARD_DEDUP_IN_FORWARD=$dif timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/d.json 2> gpurun_out/d.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/d.json') if l.startswith('{')][-1])
print('radix9=$r9 dif=$dif', d['value'], d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])
PY
done; done

mkdir -p gpurun_out
for lb in 1 2 4; do
TIERSHARD_LOOKBACK=$lb TIERSHARD_DEDUP_IN_FORWARD=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/d.json 2> gpurun_out/d.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/d.json') if l.startswith('{')][-1])
print('lookback=$lb', d['value'], d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])
PY
done

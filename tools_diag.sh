mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_table.py tests/test_plan_import.py -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/d.json 2> gpurun_out/d.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/d.json') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])
PY

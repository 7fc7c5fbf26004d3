timeout 900 python -m pytest tests/test_gpu_table.py tests/test_gpu_multigpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'], d['roofline']['frac'])"
done

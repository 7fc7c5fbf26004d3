#!/bin/bash
# Round-end check on 2 GPUs: full GPU suite (2-rank cases), smoke, N=1 A/B
# runs, then the full N=1 bench line and its ncu launch list on GPU 0.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu2.log; tail -2 gpurun_out/pytest_gpu2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
export CUDA_VISIBLE_DEVICES=0
for i in 1 2; do
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['roofline']['all_phases_ms_per_step'], d['roofline']['frac'])"
done
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench_rc=$?
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?

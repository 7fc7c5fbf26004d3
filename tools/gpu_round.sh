#!/bin/bash
# One single-GPU evidence pass (run under gpurun): GPU test suite, smoke, the
# default bench line, the reference arm, the ncu launch list and one
# ncu --set full capture per top kernel.  Outputs land in gpurun_out/.
set -u
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 16 --warmup 2 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; echo ref_rc=$?
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in gather_local seg_short piece_kernel onesweep_pass; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1; echo ncu_$k=$?
done

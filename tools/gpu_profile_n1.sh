#!/bin/bash
# N=1 profile refresh (run under gpurun on one GPU): the ncu launch list of a
# short bench run (time + DRAM bytes of every launch) and one --set full
# capture per top kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-routing"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_n1.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
for k in gather_bulk seg_short piece_kernel onesweep_pass; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1; echo ncu_$k=$?
done

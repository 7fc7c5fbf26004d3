#!/bin/bash
# NVLink + DRAM bytes per launch of the exchange kernels (run under gpurun
# --gpus N): one in-process multi-GPU probe (tools/mg_probe.py), ncu on it.
set -u
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python tools/mg_probe.py --gpus $N --steps 5 > gpurun_out/mg_probe_n$N.log 2>&1; echo probe_rc=$?; tail -2 gpurun_out/mg_probe_n$N.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
timeout 1500 ncu --metrics $M --clock-control none -k regex:"serve_rows|push_grads|replica_update|pull_requests|gather_local|seg_short|piece_kernel|long_combine|long_prefix" \
  --launch-skip $((30 * N)) --launch-count $((36 * N)) --csv --log-file gpurun_out/ncu_nvlink_n$N.csv python tools/mg_probe.py --gpus $N --steps 4 \
  > gpurun_out/ncu_nvlink_n$N.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_nvlink_n$N.log

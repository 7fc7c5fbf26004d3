#!/bin/bash
# Routing-kernel A/B + ncu capture (run under gpurun on one GPU).
set -u
mkdir -p gpurun_out
python tools/route_probe.py --topo 1x8 > gpurun_out/rp.log 2>&1
TIERSHARD_ROUTER=general python tools/route_probe.py --topo 1x8 >> gpurun_out/rp.log 2>&1
python tools/route_probe.py --topo 2x4 >> gpurun_out/rp.log 2>&1
cat gpurun_out/rp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"route_count|distinct_count" -s 4 -c 2 -o gpurun_out/prof_route_u8 python tools/route_probe.py --iters 3 > gpurun_out/ncu_route.log 2>&1; echo ncu=$?
timeout 300 python -m pytest tests/test_gpu_router.py -q -x 2>&1 | tail -2

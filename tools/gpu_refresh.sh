#!/bin/bash
# Short end-of-round confirmation (run under gpurun on one GPU): smoke, the
# default N=1 bench line, then the GPU test suite.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/refresh_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/refresh_smoke.log
timeout 240 python bench.py > gpurun_out/refresh_bench_n1.json 2> gpurun_out/refresh_bench_n1.err; echo bench_rc=$?
timeout 420 python -m pytest tests -q -m gpu -x > gpurun_out/refresh_pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/refresh_pytest_gpu.log

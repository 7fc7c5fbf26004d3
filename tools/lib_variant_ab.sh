#!/bin/bash
# A/B of library build variants (paper_2301_02959_b200/lib/variants/*.so,
# built with NVFLAGS_EXTRA): each is swapped in, checked by the one-GPU
# table tests, and timed by the N-GPU bench.  bash tools/lib_variant_ab.sh N v1 v2 ...
set -u
N=$1; shift
mkdir -p gpurun_out
L=paper_2301_02959_b200/lib
cp $L/libtiershard_b200.so $L/variants/_orig.so
: > gpurun_out/lib_ab.txt
for v in "$@"; do
  cp $L/variants/$v.so $L/libtiershard_b200.so
  timeout 300 python -m pytest tests/test_gpu_table.py -q -x > gpurun_out/lib_ab_pytest.log 2>&1; rc=$?
  if [ "$N" = "1" ]; then
    timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-routing > gpurun_out/ab.json 2> gpurun_out/ab.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  fi
  tail -1 gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v tests_rc=$rc', d['ms_per_step'], d['roofline']['all_phases_ms_per_step'])" >> gpurun_out/lib_ab.txt 2>&1
done
cp $L/variants/_orig.so $L/libtiershard_b200.so
cat gpurun_out/lib_ab.txt

#!/bin/bash
# Register gather vs bulk-copy (cp.async.bulk) gather on one GPU: parity
# tests under the bulk variant, then the N=1 bench step for each grid, then
# one ncu capture of each kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
[ -z "${GAB_SKIP_TESTS:-}" ] && TIERSHARD_GATHER=bulk timeout 600 python -m pytest tests/test_gpu_table.py -q -x > gpurun_out/gab_pytest.log 2>&1; echo bulk_pytest_rc=$?; tail -1 gpurun_out/gab_pytest.log
B="python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-routing"
: > gpurun_out/gather_ab.txt
if [ $# -eq 0 ]; then set -- "reg 6 4" "bulk 2 4" "bulk 3 4" "reg 8 4"; fi
for v in "$@"; do
  set -- $v
  if [ "$1" = "bulk" ]; then G=bulk; else G=reg; fi
  env TIERSHARD_GATHER=$G TIERSHARD_GATHER_BLOCKS=$2 TIERSHARD_BULK_STAGES=$3 ${4:-} timeout 600 $B > gpurun_out/gab.json 2> gpurun_out/gab.err
  tail -1 gpurun_out/gab.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$1 blocks/SM=$2 stages=$3', d['ms_per_step'], 'gather', r['all_phases_ms_per_step'].get('gather'), 'gbs', r.get('gather_gbs'), 'sort', r['all_phases_ms_per_step'].get('dedup_sort'), 'fwd', d['lookup_exchange']['ms_per_forward'])" >> gpurun_out/gather_ab.txt 2>&1
done
cat gpurun_out/gather_ab.txt
P="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-routing"
[ -z "${GAB_SKIP_NCU:-}" ] && TIERSHARD_GATHER=bulk TIERSHARD_GATHER_BLOCKS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_bulk -s 2 -c 1 -o gpurun_out/prof_gather_bulk $P > gpurun_out/ncu_gab.log 2>&1; echo ncu=$?

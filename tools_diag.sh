mkdir -p gpurun_out
run() {  # tag env...
tag=$1; shift
env "$@" TS_BENCH_DIAG=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 20 --warmup 5 --tables 16 --rows 25000000 --seq-len 256 --virtual-nodes --sampler gpu --no-e2e \
  --cache /tmp/c4cache > gpurun_out/c4_$tag.json 2> gpurun_out/c4_$tag.err
python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/c4_$tag.json') if l.startswith('{')][-1])
print('$tag', d['value'], d['ms_per_step'], d['step_ms_min_median_max_rank0'], d['nvlink']['achieved_gbs'])
print('  ', d['roofline']['all_phases_ms_per_step'])
PY
}
run base
run push4 TIERSHARD_PUSH_BLOCKS=4
run serve192 TIERSHARD_SERVE_BLOCKS=192
run both TIERSHARD_PUSH_BLOCKS=4 TIERSHARD_SERVE_BLOCKS=192

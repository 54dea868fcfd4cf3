#!/bin/bash
# Multi-GPU measurement plan (needs >= 2 GPUs on one node; not runnable in a
# 1-GPU pool): bitwise checks of every decomposition and transport, then the
# cfg-5 strong-scaling bench lines with both z-slab transports.
#   bash tools/gpu_scaling.sh [max_gpus]
set -u
MAX=${1:-8}
mkdir -p gpurun_out/scaling
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4 8; do
  [ "$n" -le "$MAX" ] || continue
  for name in aa-soa blk-push-soa blk-pull-soa; do
    for tr in peer copy; do
      timeout 900 $R --nproc-per-node $n --master-port $((29500 + n)) tools/mgpu_check.py 64 32 48 10 channel $name $tr \
        > gpurun_out/scaling/check_${n}_${name}_${tr}.log 2>&1
    done
  done
  timeout 900 $R --nproc-per-node $n --master-port $((29600 + n)) tools/mgpu_check.py 64 32 48 10 channel list-aa-soa copy \
    > gpurun_out/scaling/check_${n}_list.log 2>&1
done
timeout 900 python bench.py > gpurun_out/scaling/bench_1.json 2> gpurun_out/scaling/bench_1.err
for n in 2 4 8; do
  [ "$n" -le "$MAX" ] || continue
  for tr in peer copy; do
    timeout 900 $R --nproc-per-node $n --master-port $((29700 + n)) bench.py --gpus $n --transport $tr \
      > gpurun_out/scaling/bench_${n}_${tr}.json 2> gpurun_out/scaling/bench_${n}_${tr}.err
  done
done
grep -h "PASS\|FAIL" gpurun_out/scaling/check_*.log

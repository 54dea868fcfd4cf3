#!/bin/bash
# cfg 1 fused: arithmetic target test in push; shapes 1/3/4 for push, pull, aa
mkdir -p gpurun_out
for k in blk-push-soa blk-pull-soa aa-soa blk-push-aos; do for sh in 1 3 4; do
LBMGPU_FUSED_SHAPE=$sh timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b28_${k}_$sh.json 2>&1; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle_steppers or flow_launch or fingerprint" > gpurun_out/p28.log 2>&1; echo pytest rc=$? >> gpurun_out/p28.log

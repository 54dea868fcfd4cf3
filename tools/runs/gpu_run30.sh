#!/bin/bash
# two-level grid barrier: parity + cfg 1 kinds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle_steppers or flow_launch or fingerprint or poiseuille" > gpurun_out/p30.log 2>&1; echo pytest rc=$? >> gpurun_out/p30.log
for k in blk-push-soa blk-pull-soa aa-soa; do for i in 1 2; do
timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b30_${k}_$i.json 2>&1; done; done

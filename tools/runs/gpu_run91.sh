#!/bin/bash
mkdir -p gpurun_out/r91
for k in blk-push-soa blk-pull-soa aa-soa; do
  for sh in -1 6 7 8; do
    LBMGPU_FUSED_SHAPE=$sh timeout 300 python bench.py --config 1 --kernel $k --steps 100 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r91/${k}_s$sh.json 2> gpurun_out/r91/${k}_s$sh.err
  done
done

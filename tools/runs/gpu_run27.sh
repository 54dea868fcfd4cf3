#!/bin/bash
# cfg 1 grid-barrier kernel block shapes
mkdir -p gpurun_out
for sh in 0 5 1 2 3 4 0; do LBMGPU_FUSED_SHAPE=$sh timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b27_sh$sh.json 2> gpurun_out/b27_sh$sh.err; done
LBMGPU_FUSED_SHAPE=0 timeout 120 python bench.py --config 1 --kernel blk-pull-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b27_pull0.json 2>&1
LBMGPU_FUSED_SHAPE=3 timeout 120 python bench.py --config 1 --kernel blk-pull-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b27_pull3.json 2>&1
LBMGPU_FUSED_SHAPE=0 timeout 120 python bench.py --config 1 --kernel aa-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b27_aa0.json 2>&1
LBMGPU_FUSED_SHAPE=3 timeout 120 python bench.py --config 1 --kernel aa-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b27_aa3.json 2>&1

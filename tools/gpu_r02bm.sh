#!/bin/bash
# Round 2bm: ncu --set full (with source) of the cfg-1 fused push launch
mkdir -p gpurun_out
CMD="python bench.py --config 1 --steps 20 --warmup 0 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/r02bm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_full_fused -c 1 -o gpurun_out/r02bm_c1_fused $CMD > gpurun_out/r02bm_ncu.log 2>&1
echo ncu rc=$?

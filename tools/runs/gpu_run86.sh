#!/bin/bash
# ncu --set full of the cfg-1 fused push (stall reasons, source counters)
mkdir -p gpurun_out/r86
C="python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$C > gpurun_out/r86/plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/r86/c1_push $C > gpurun_out/r86/ncu.log 2>&1; echo rc=$? >> gpurun_out/r86/ncu.log

#!/bin/bash
mkdir -p gpurun_out
C="python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$C > gpurun_out/r01g_plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/r01g_prof_c1 $C > gpurun_out/r01g_ncu_c1.log 2>&1; echo c1 rc=$?

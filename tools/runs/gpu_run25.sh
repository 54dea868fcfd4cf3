#!/bin/bash
# cfg 1 fused push: full ncu capture (one launch = 4 sweeps) + e2e check on cfg 5
mkdir -p gpurun_out
B="python bench.py --config 1 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/b25_c1.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/r25_fused $B > gpurun_out/r25_ncu.log 2>&1; echo ncu rc=$?
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-micro > gpurun_out/b25_c5.json 2> gpurun_out/b25_c5.err

#!/bin/bash
# Round 2bt: ncu --set full (with source) of the list AoS pull tile kernel on cfg 2
mkdir -p gpurun_out
CMD="python bench.py --config 2 --kernel list-pull-aos --steps 4 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/r02bt_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_list_pull_aos_tile -s 2 -c 1 -o gpurun_out/r02bt_list_pull_aos $CMD > gpurun_out/r02bt_ncu.log 2>&1
echo ncu rc=$?

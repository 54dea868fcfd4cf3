#!/bin/bash
# Round 2bk: ncu --set full (with source) of the list AoS AA odd staging-tile kernel on cfg 2
mkdir -p gpurun_out
CMD="python bench.py --config 2 --kernel list-aa-aos --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/r02bk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_list_aa_odd_aos_tile -s 1 -c 1 -o gpurun_out/r02bk_list_aa_aos $CMD > gpurun_out/r02bk_ncu.log 2>&1
echo ncu rc=$?

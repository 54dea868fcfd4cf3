#!/bin/bash
# Round 2az: ncu --set full of the round-2 AoS tile kernels (one launch each)
TAG=${1:-r02az}
mkdir -p gpurun_out
run() {  # name cfg kernel-regex extra
  CMD="python bench.py --config $2 --kernel $1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro $4"
  $CMD > gpurun_out/${TAG}_$1_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o gpurun_out/${TAG}_$1 $CMD > gpurun_out/${TAG}_$1_ncu.log 2>&1
  echo $1 ncu rc=$?
}
run list-aa-aos 2 k_list_aa_odd_aos_tile ""
run aa-aos 5 k_full_aa_odd_aos_tile3d "--dims 1024x512x64"
run blk-pull-aos 5 k_full_pull_aos_tile3d "--dims 1024x512x64"

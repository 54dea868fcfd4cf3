#!/bin/bash
# L2-capacity probe for the fused (L2-resident) multi-sweep launches: MFLUP/s and ncu DRAM bytes vs lattice size
mkdir -p gpurun_out/r66
for spec in "blk-push-soa 64x64x32" "blk-push-soa 64x64x48" "blk-push-soa 64x64x56" "blk-push-soa 64x64x64" "blk-push-soa 64x64x72" \
            "aa-soa 64x64x64" "aa-soa 64x64x96" "aa-soa 64x64x128" "aa-soa 64x64x144"; do
  set -- $spec
  tag=$1_$2
  timeout 300 python bench.py --config 1 --kernel $1 --dims $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r66/$tag.json 2> gpurun_out/r66/$tag.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:fused -c 2 --csv \
     python bench.py --config 1 --kernel $1 --dims $2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r66/$tag.ncu.csv 2> gpurun_out/r66/$tag.ncu.err
done

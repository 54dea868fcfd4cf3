#!/bin/bash
# AoS and the other names on the BASELINE geometries
mkdir -p gpurun_out
for k in aa-aos aa-soa aa-vec-soa blk-push-aos blk-pull-aos blk-pull-soa; do
timeout 300 python bench.py --config 5 --kernel $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b33_c5_$k.json 2>&1; done
for k in list-aa-aos list-pull-aos list-push-soa list-push-aos list-aa-pv-soa list-pull-split-nt-1s-soa; do
timeout 300 python bench.py --config 2 --kernel $k --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b33_c2_$k.json 2>&1; done

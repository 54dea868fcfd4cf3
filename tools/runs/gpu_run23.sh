#!/bin/bash
# AA CTA size sweep on cfg 5
mkdir -p gpurun_out
for t in 256 128 64 256; do LBMGPU_AA_THREADS=$t timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b23_t$t.json 2> gpurun_out/b23_t$t.err; done

#!/bin/bash
# list CTA size sweep (cfg 2/3/4, ria), AA default now 128
mkdir -p gpurun_out
for t in 256 128; do
  LBMGPU_LIST_THREADS=$t timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --kernel list-aa-ria-soa > gpurun_out/b24_c2_t$t.json 2> gpurun_out/b24_c2_t$t.err
  LBMGPU_LIST_THREADS=$t timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b24_c3_t$t.json 2> gpurun_out/b24_c3_t$t.err
  LBMGPU_LIST_THREADS=$t timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b24_c4_t$t.json 2> gpurun_out/b24_c4_t$t.err
done
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b24_c5.json 2> gpurun_out/b24_c5.err

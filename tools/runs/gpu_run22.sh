#!/bin/bash
# odd-step constant-offset fast path: parity + cfg 5 bench (x2) + cfg 4/2 (blocks wrap paths)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "aa or zslab or fused or smoke" > gpurun_out/p22.log 2>&1; echo pytest rc=$? >> gpurun_out/p22.log
for i in 1 2; do timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b22_c5_$i.json 2> gpurun_out/b22_c5_$i.err; done


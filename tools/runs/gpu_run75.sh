#!/bin/bash
# e2e with the transfer-path warm-up: cfg 1 and cfg 5
mkdir -p gpurun_out/r75
timeout 300 python bench.py --config 1 --no-cpu-baseline --no-micro > gpurun_out/r75/c1.json 2> gpurun_out/r75/c1.err
timeout 600 python bench.py --no-cpu-baseline --no-micro > gpurun_out/r75/c5.json 2> gpurun_out/r75/c5.err

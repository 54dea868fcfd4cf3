#!/bin/bash
mkdir -p gpurun_out/r81
timeout 900 python bench.py --config 1 --steps 100 > gpurun_out/r81/cfg1_100.json 2> gpurun_out/r81/cfg1_100.err
timeout 900 python bench.py --config 1 > gpurun_out/r81/cfg1_20.json 2> gpurun_out/r81/cfg1_20.err

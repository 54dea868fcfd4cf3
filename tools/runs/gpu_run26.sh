#!/bin/bash
# dataflow fused kernel: parity, then cfg 1 bench flow 256/128 vs grid barrier
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle_steppers or flow_launch or fingerprint or poiseuille" > gpurun_out/p26.log 2>&1; echo pytest rc=$? >> gpurun_out/p26.log
for f in 256 128 0 256 64; do LBMGPU_FUSED_FLOW=$f timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b26_c1_f$f.json 2> gpurun_out/b26_c1_f$f.err; done
LBMGPU_FUSED_FLOW=256 timeout 120 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b26_c1_s100.json 2>&1

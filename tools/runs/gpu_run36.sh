#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or edge or oracle_steppers or node_range or poiseuille_every" > gpurun_out/p36.log 2>&1; echo pytest rc=$? >> gpurun_out/p36.log
for k in aa-aos blk-pull-aos blk-push-aos; do timeout 300 python bench.py --config 5 --kernel $k --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b36_c5_$k.json 2>&1; done
for k in list-aa-aos list-pull-aos; do timeout 300 python bench.py --config 2 --kernel $k --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b36_c2_$k.json 2>&1; done

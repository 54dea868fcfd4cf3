#!/bin/bash
# cfg 1 fused push: two nodes per thread and round (shapes 6-9) vs the default (3); parity first
mkdir -p gpurun_out/r68
for sh in 6 7 8 9; do
  LBMGPU_FUSED_SHAPE=$sh timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or push" > gpurun_out/r68/pytest_$sh.log 2>&1; echo rc=$? >> gpurun_out/r68/pytest_$sh.log
done
for sh in 3 6 7 8 9; do
  for st in 20 100; do
    LBMGPU_FUSED_SHAPE=$sh timeout 300 python bench.py --config 1 --steps $st --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r68/c1_s${sh}_${st}.json 2> gpurun_out/r68/c1_s${sh}_${st}.err
  done
done

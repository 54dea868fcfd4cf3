#!/bin/bash
# fused push with L1-cached loads + next-node L1 prefetch (experiment): parity (repeated), cfg 1
mkdir -p gpurun_out/r96
for i in 1 2 3; do
LBMGPU_FUSED_L1=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "push or fused or randomized or baseline_config_fingerprint and not alternative" > gpurun_out/r96/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r96/pytest_$i.log
done
for l1 in 0 1; do
  for st in 20 100; do
    LBMGPU_FUSED_L1=$l1 timeout 300 python bench.py --config 1 --steps $st --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r96/c1_l1${l1}_$st.json 2> gpurun_out/r96/c1_l1${l1}_$st.err
  done
done

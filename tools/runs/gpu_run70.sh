#!/bin/bash
# RIA pattern-id odd step register variants (LBMGPU_RIA_PID_VARIANT 0-4), cfg 4 and cfg 2
mkdir -p gpurun_out/r70
for v in 0 1 2 3 4; do
  LBMGPU_RIA_PID_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ria_pattern_id_widths or ria_codings" > gpurun_out/r70/pytest_$v.log 2>&1; echo rc=$? >> gpurun_out/r70/pytest_$v.log
  for c in 4 2; do
    LBMGPU_RIA_PID_VARIANT=$v timeout 300 python bench.py --config $c --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r70/c${c}_v$v.json 2> gpurun_out/r70/c${c}_v$v.err
  done
done

#!/bin/bash
# peer AA path with the boundary work on its own stream: parity (repeated, concurrency), emulated probe
mkdir -p gpurun_out/r83
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "peer" > gpurun_out/r83/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r83/pytest_$i.log
done
timeout 900 python tools/fuzz_parity.py 300 80000 > gpurun_out/r83/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r83/fuzz.log
for parts in 2 8; do
  for tr in copy peer; do
    timeout 300 python bench.py --virtual-parts $parts --transport $tr --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r83/vp${parts}_${tr}.json 2> gpurun_out/r83/vp${parts}_${tr}.err
  done
done

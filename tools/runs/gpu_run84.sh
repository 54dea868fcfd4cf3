#!/bin/bash
# one-step peer path with the boundary stream: parity (repeated), fuzz, emulated probe
mkdir -p gpurun_out/r84
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "peer" > gpurun_out/r84/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r84/pytest_$i.log
done
timeout 900 python tools/fuzz_parity.py 300 90000 > gpurun_out/r84/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r84/fuzz.log
for k in blk-push-soa blk-pull-soa; do
  for tr in copy peer; do
    timeout 300 python bench.py --kernel $k --virtual-parts 8 --transport $tr --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r84/${k}_vp8_$tr.json 2> gpurun_out/r84/${k}_vp8_$tr.err
  done
done

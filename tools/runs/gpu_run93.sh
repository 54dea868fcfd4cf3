#!/bin/bash
# one-step copy-halo path with the boundary stream: parity (repeated), fuzz, emulated probe
mkdir -p gpurun_out/r93
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "zslab or guard or alternative" > gpurun_out/r93/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r93/pytest_$i.log
done
timeout 900 python tools/fuzz_parity.py 300 96000 > gpurun_out/r93/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r93/fuzz.log
for k in blk-push-soa blk-pull-soa; do
  timeout 300 python bench.py --kernel $k --virtual-parts 8 --transport copy --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r93/${k}_vp8_copy.json 2> gpurun_out/r93/${k}_vp8_copy.err
done

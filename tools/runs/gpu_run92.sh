#!/bin/bash
# copy-halo AA path with the boundary stream: parity (repeated), fuzz, emulated probe
mkdir -p gpurun_out/r92
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "zslab or guard or alternative" > gpurun_out/r92/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r92/pytest_$i.log
done
timeout 900 python tools/fuzz_parity.py 300 95000 > gpurun_out/r92/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r92/fuzz.log
for parts in 2 8; do
  timeout 300 python bench.py --virtual-parts $parts --transport copy --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r92/vp${parts}_copy.json 2> gpurun_out/r92/vp${parts}_copy.err
  timeout 300 python bench.py --virtual-parts $parts --transport copy --nccl-self --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r92/vp${parts}_nccl.json 2> gpurun_out/r92/vp${parts}_nccl.err
done

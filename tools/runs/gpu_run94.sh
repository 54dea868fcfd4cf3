#!/bin/bash
# list node-range parts with the boundary stream: parity (repeated), fuzz, emulated probe
mkdir -p gpurun_out/r94
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "list_node_range or list_parts or guard or local_rows" > gpurun_out/r94/pytest_$i.log 2>&1; echo rc=$? >> gpurun_out/r94/pytest_$i.log
done
timeout 900 python tools/fuzz_parity.py 300 97000 > gpurun_out/r94/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r94/fuzz.log
for parts in 2 8; do
  timeout 300 python bench.py --config 2 --virtual-parts $parts --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r94/c2_vp$parts.json 2> gpurun_out/r94/c2_vp$parts.err
done

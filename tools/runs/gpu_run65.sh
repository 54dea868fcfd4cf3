#!/bin/bash
# peer-memory transport: parity tests, then the cfg-5 emulated decomposition probe (copy vs peer)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "peer or zslab" > gpurun_out/r65_pytest.log 2>&1; echo rc=$? >> gpurun_out/r65_pytest.log
for parts in 2 8; do
  for tr in copy peer; do
    timeout 300 python bench.py --virtual-parts $parts --transport $tr --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r65_vp${parts}_${tr}.json 2> gpurun_out/r65_vp${parts}_${tr}.err
  done
done

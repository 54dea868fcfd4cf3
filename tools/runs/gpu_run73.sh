#!/bin/bash
# peer transport for the one-step push / pull z slabs: parity, C++ API test, emulated probes
mkdir -p gpurun_out/r73
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_api.py -q -x -k "peer or zslab or cpp" > gpurun_out/r73/pytest.log 2>&1; echo rc=$? >> gpurun_out/r73/pytest.log
for k in blk-push-soa blk-pull-soa; do
  for tr in copy peer; do
    timeout 300 python bench.py --kernel $k --virtual-parts 8 --transport $tr --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r73/${k}_vp8_$tr.json 2> gpurun_out/r73/${k}_vp8_$tr.err
  done
done
timeout 900 python tools/fuzz_parity.py 400 60000 > gpurun_out/r73/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r73/fuzz.log

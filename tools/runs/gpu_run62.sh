#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b62.txt
LBMGPU_L2_HINTS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "flow_launch and push" > gpurun_out/p62.log 2>&1; echo rc=$? >> gpurun_out/p62.log
for h in 0 1 0 1; do
LBMGPU_L2_HINTS=$h timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hints $h', round(d['value']))" >> gpurun_out/b62.txt
done

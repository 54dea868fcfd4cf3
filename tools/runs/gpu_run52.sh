#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b52.txt
LBMGPU_GRID_SYNC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "flow_launch or oracle_steppers" > gpurun_out/p52.log 2>&1; echo rc=$? >> gpurun_out/p52.log
for m in 0 1 0 1; do for k in blk-push-soa blk-pull-soa aa-soa; do
LBMGPU_GRID_SYNC=$m timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sync', $m, '$k', round(d['value']))" >> gpurun_out/b52.txt
done; done

#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b53.txt
for sh in 1 3 4 0 5; do for k in blk-push-soa blk-pull-soa aa-soa; do
LBMGPU_FUSED_SHAPE=$sh timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shape', $sh, '$k', round(d['value']))" >> gpurun_out/b53.txt
done; done

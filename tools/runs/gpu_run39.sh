#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b39.txt
for f in 0 256 128; do for k in blk-push-soa blk-pull-soa aa-soa; do
LBMGPU_FUSED_FLOW=$f timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flow', $f, '$k', round(d['value']))" >> gpurun_out/b39.txt
done; done

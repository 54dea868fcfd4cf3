#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b50.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "flow" > gpurun_out/p50.log 2>&1; echo rc=$? >> gpurun_out/p50.log
for f in 0 320 160 128; do for k in blk-push-soa blk-pull-soa aa-soa; do
LBMGPU_FUSED_FLOW=$f timeout 120 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flow', $f, '$k', round(d['value']))" >> gpurun_out/b50.txt
done; done

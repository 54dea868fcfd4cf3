#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b63.txt
for i in 1 2; do
timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['value']))" >> gpurun_out/b63.txt
done

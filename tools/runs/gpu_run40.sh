#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "node_range or list_parts or local_rows or zslab" > gpurun_out/p40.log 2>&1; echo pytest rc=$? >> gpurun_out/p40.log
for vp in 1 2 4 8; do timeout 300 python bench.py --config 2 --virtual-parts $vp --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($vp, round(d['value']))" >> gpurun_out/b40.txt; done

#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b60.txt
for st in 0 12 3 4; do
LBMGPU_AA_TMA_STAGES=$st timeout 300 python bench.py --config 5 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma $st', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b60.txt
done

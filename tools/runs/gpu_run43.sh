#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b43.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "zslab_parts and aa-soa" > gpurun_out/p43.log 2>&1; echo rc=$? >> gpurun_out/p43.log
for w in 0 0.5 1 2 4 0; do
LBMGPU_AA_PF_WAVES=$w timeout 300 python bench.py --config 5 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b43.txt
done

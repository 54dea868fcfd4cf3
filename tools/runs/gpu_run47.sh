#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b47.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "halo_tiles or golden or edge" > gpurun_out/p47.log 2>&1; echo rc=$? >> gpurun_out/p47.log
for t in 1 0; do
LBMGPU_ODD_TILE=$t timeout 300 python bench.py --config 5 --kernel aa-aos --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile $t', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b47.txt
done

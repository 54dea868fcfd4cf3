#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b44.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or edge or oracle_steppers" > gpurun_out/p44.log 2>&1; echo rc=$? >> gpurun_out/p44.log
for t in 1 0; do for band in 16 0; do
LBMGPU_AOS_TILE=$t LBMGPU_AOS_BAND=$band timeout 300 python bench.py --config 5 --kernel blk-push-aos --dims 1024x512x128 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile $t band $band', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b44.txt
done; done

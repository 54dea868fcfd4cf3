#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "realigned" > gpurun_out/p34.log 2>&1; echo pytest rc=$? >> gpurun_out/p34.log
for sx in 0 4 3 0 4; do LBMGPU_AA_ODD_SX=$sx timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b34_sx$sx.json 2>&1; cat gpurun_out/b34_sx$sx.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($sx, round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b34.txt; done

#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b41.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ria or golden or edge" > gpurun_out/p41.log 2>&1; echo pytest rc=$? >> gpurun_out/p41.log
for c in 2 4; do for m in 0 2 -1; do
LBMGPU_RIA_MODE=$m timeout 300 python bench.py --config $c --kernel list-aa-ria-soa --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>gpurun_out/b41_err_$c_$m.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, $m, round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b41.txt
done; done

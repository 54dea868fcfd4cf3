#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b49.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/p49.log 2>&1; echo rc=$? >> gpurun_out/p49.log
for c in 5 2 4; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b49.txt; done

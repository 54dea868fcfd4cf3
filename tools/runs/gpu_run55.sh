#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b55.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "flow_launch or oracle_steppers or golden or poiseuille or baseline_config" > gpurun_out/p55.log 2>&1; echo rc=$? >> gpurun_out/p55.log
for i in 1 2; do timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 default', round(d['value']), d['roofline']['frac'])" >> gpurun_out/b55.txt; done
timeout 120 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 K=100', round(d['value']), d['roofline']['frac'])" >> gpurun_out/b55.txt

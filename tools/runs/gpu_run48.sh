#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b48.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cli.py tests/test_cpp_api.py -q -x -k "golden or oracle_steppers or local_rows or baseline_config or cli or cpp" > gpurun_out/p48.log 2>&1; echo rc=$? >> gpurun_out/p48.log
for c in 1 2 5; do timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, round(d['value']), d['e2e'])" >> gpurun_out/b48.txt; done

#!/bin/bash
mkdir -p gpurun_out/r82
timeout 1200 python tools/fuzz_parity.py 600 70000 > gpurun_out/r82/fuzz.log 2>&1; echo rc=$? >> gpurun_out/r82/fuzz.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or temporal" > gpurun_out/r82/pytest.log 2>&1; echo rc=$? >> gpurun_out/r82/pytest.log
for i in 1 2 3; do timeout 300 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r82/cfg1_$i.json 2> gpurun_out/r82/cfg1_$i.err; done

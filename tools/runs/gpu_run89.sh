#!/bin/bash
# list pull through Gather-table pattern ids: parity, cfg 3 bench
mkdir -p gpurun_out/r89
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pull_pattern" > gpurun_out/r89/pytest.log 2>&1; echo rc=$? >> gpurun_out/r89/pytest.log
B="python bench.py --config 3 --no-e2e --no-cpu-baseline --no-micro"
timeout 600 $B > gpurun_out/r89/c3.json 2> gpurun_out/r89/c3.err
LBMGPU_PULL_PID=1 timeout 600 $B > gpurun_out/r89/c3_pid.json 2> gpurun_out/r89/c3_pid.err
LBMGPU_PULL_PID=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_fingerprint and 3 and not alternative" > gpurun_out/r89/golden.log 2>&1; echo rc=$? >> gpurun_out/r89/golden.log

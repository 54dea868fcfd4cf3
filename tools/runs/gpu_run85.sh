#!/bin/bash
mkdir -p gpurun_out/r85
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_fingerprint" --durations=12 > gpurun_out/r85/pytest.log 2>&1; echo rc=$? >> gpurun_out/r85/pytest.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "randomized" > gpurun_out/p64.log 2>&1; echo rc=$? >> gpurun_out/p64.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "list_fused_launch" > gpurun_out/p58.log 2>&1; echo rc=$? >> gpurun_out/p58.log

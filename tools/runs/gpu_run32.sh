#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "edge" > gpurun_out/p32.log 2>&1; echo pytest rc=$? >> gpurun_out/p32.log

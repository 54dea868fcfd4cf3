#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "zslab or local_rows" > gpurun_out/p31.log 2>&1; echo pytest rc=$? >> gpurun_out/p31.log

#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "node_range" > gpurun_out/p51.log 2>&1; echo rc=$? >> gpurun_out/p51.log

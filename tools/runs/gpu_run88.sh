#!/bin/bash
mkdir -p gpurun_out/r88
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "guard" > gpurun_out/r88/pytest.log 2>&1; echo rc=$? >> gpurun_out/r88/pytest.log

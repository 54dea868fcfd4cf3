#!/bin/bash
# final: every GPU test incl. the slow full-size extras
mkdir -p gpurun_out/r95
LBMGPU_SLOW=1 timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r95/pytest_slow.log 2>&1; echo rc=$? >> gpurun_out/r95/pytest_slow.log

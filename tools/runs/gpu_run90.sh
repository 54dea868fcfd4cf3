#!/bin/bash
# final check of round 1h: every GPU test incl. the slow full-size extras, then the round-end script
mkdir -p gpurun_out/r90
LBMGPU_SLOW=1 timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r90/pytest_slow.log 2>&1; echo rc=$? >> gpurun_out/r90/pytest_slow.log
bash tools/gpu_roundend.sh

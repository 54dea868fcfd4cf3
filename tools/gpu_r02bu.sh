#!/bin/bash
# Round 2bu: guard-zone test with the interior AoS tiles and the pipelined job, ncu traffic capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "guard" 2>&1 | tail -2
bash tools/gpu_ncu_summary.sh

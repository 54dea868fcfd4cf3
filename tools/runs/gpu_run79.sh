#!/bin/bash
mkdir -p gpurun_out/r79
timeout 600 python -m pytest tests/test_peer_ipc.py tests/test_gpu_parity.py -q -x -k "peer" -rs > gpurun_out/r79/pytest.log 2>&1; echo rc=$? >> gpurun_out/r79/pytest.log

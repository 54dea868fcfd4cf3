#!/bin/bash
mkdir -p gpurun_out/r87
timeout 600 python -m pytest tests/test_peer_ipc.py -q -x > gpurun_out/r87/pytest.log 2>&1; echo rc=$? >> gpurun_out/r87/pytest.log

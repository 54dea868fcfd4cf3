#!/bin/bash
# parity fuzzing incl. the peer transport and every RIA coding (random RIA_MODE)
mkdir -p gpurun_out
timeout 1500 python tools/fuzz_parity.py 600 40000 > gpurun_out/r71_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r71_fuzz.log
FUZZ_BIG=1 timeout 1200 python tools/fuzz_parity.py 200 50000 > gpurun_out/r71_fuzz_big.log 2>&1; echo rc=$? >> gpurun_out/r71_fuzz_big.log

#!/bin/bash
# Round 2bp: fuzz parity on the final sources (after the AoS tile fast path and the 32-bit fused indices)
mkdir -p gpurun_out
timeout 1500 python tools/fuzz_parity.py 600 151000 > gpurun_out/r02bp_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r02bp_fuzz.log
FUZZ_BIG=1 timeout 900 python tools/fuzz_parity.py 60 157000 > gpurun_out/r02bp_fuzz_big.log 2>&1; echo rc=$? >> gpurun_out/r02bp_fuzz_big.log
tail -n 2 gpurun_out/r02bp_fuzz.log; tail -n 2 gpurun_out/r02bp_fuzz_big.log

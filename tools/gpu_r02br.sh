#!/bin/bash
# Round 2br: large fuzz parity run on the final sources
mkdir -p gpurun_out
timeout 2400 python tools/fuzz_parity.py 3000 171000 > gpurun_out/r02br_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r02br_fuzz.log
FUZZ_BIG=1 timeout 2400 python tools/fuzz_parity.py 400 177000 > gpurun_out/r02br_fuzz_big.log 2>&1; echo rc=$? >> gpurun_out/r02br_fuzz_big.log
tail -n 2 gpurun_out/r02br_fuzz.log; tail -n 2 gpurun_out/r02br_fuzz_big.log

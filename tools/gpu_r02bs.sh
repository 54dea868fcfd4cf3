#!/bin/bash
# Round 2bs: large fuzz parity run with the AoS interior-tile cases
mkdir -p gpurun_out
timeout 2400 python tools/fuzz_parity.py 2000 181000 > gpurun_out/r02bs_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r02bs_fuzz.log
FUZZ_BIG=1 timeout 2400 python tools/fuzz_parity.py 300 187000 > gpurun_out/r02bs_fuzz_big.log 2>&1; echo rc=$? >> gpurun_out/r02bs_fuzz_big.log
tail -n 2 gpurun_out/r02bs_fuzz.log; tail -n 2 gpurun_out/r02bs_fuzz_big.log

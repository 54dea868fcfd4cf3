#!/bin/bash
# Round 2bi: fuzz parity on the final sources (new seeds), then the round-end rehearsal
mkdir -p gpurun_out
timeout 1500 python tools/fuzz_parity.py 500 131000 > gpurun_out/r02bi_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r02bi_fuzz.log
FUZZ_BIG=1 timeout 900 python tools/fuzz_parity.py 60 137000 > gpurun_out/r02bi_fuzz_big.log 2>&1; echo rc=$? >> gpurun_out/r02bi_fuzz_big.log
tail -2 gpurun_out/r02bi_fuzz.log gpurun_out/r02bi_fuzz_big.log
bash tools/gpu_roundend.sh

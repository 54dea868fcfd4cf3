#!/bin/bash
# cfg 1 push: target mask vs flags, fused shapes 1/3, per-sweep
mkdir -p gpurun_out
for tm in 1 0; do for sh in 1 3; do
LBMGPU_PUSH_TMASK=$tm LBMGPU_FUSED_SHAPE=$sh timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b29_tm${tm}_$sh.json 2>&1; done
LBMGPU_PUSH_TMASK=$tm LBMGPU_FUSED_MB=0 timeout 120 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b29_tm${tm}_ps.json 2>&1
LBMGPU_PUSH_TMASK=$tm timeout 120 python bench.py --config 5 --kernel blk-push-soa --steps 4 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b29_tm${tm}_c5.json 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle_steppers or flow_launch or fingerprint or golden" > gpurun_out/p29.log 2>&1; echo pytest rc=$? >> gpurun_out/p29.log

#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b54.txt
for sh in 5 3; do
LBMGPU_FUSED_SHAPE=$sh timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "flow_launch or oracle_steppers or golden" > gpurun_out/p54_$sh.log 2>&1; echo rc=$? >> gpurun_out/p54_$sh.log
done
for sh in 5 3 5; do for k in aa-soa aa-aos blk-pull-soa; do
LBMGPU_FUSED_SHAPE=$sh timeout 120 python bench.py --config 1 --kernel $k --steps 100 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shape', $sh, '$k', round(d['value']), d['ms_per_step'])" >> gpurun_out/b54.txt
done; done

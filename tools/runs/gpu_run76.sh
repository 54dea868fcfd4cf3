#!/bin/bash
# push / pull warp-uniform fast paths: parity, cfg 1 fused, cfg-5 box per-sweep
mkdir -p gpurun_out/r76
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "push or pull or randomized or fused or zslab" > gpurun_out/r76/pytest.log 2>&1; echo rc=$? >> gpurun_out/r76/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --no-micro"
for k in blk-push-soa blk-pull-soa; do
  timeout 300 $B --config 1 --kernel $k --steps 100 > gpurun_out/r76/c1_$k.json 2> gpurun_out/r76/c1_$k.err
  timeout 300 $B --kernel $k > gpurun_out/r76/c5box_$k.json 2> gpurun_out/r76/c5box_$k.err
done
timeout 300 $B --config 1 --steps 20 > gpurun_out/r76/c1_default.json 2> gpurun_out/r76/c1_default.err

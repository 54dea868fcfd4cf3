#!/bin/bash
# CUDA-graph replay of the per-sweep launches: parity, then cfg 1 / 96^3 / cfg 5 with and without graphs
mkdir -p gpurun_out/r74
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "graph" > gpurun_out/r74/pytest.log 2>&1; echo rc=$? >> gpurun_out/r74/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --no-micro"
for g in 0 1; do
  LBMGPU_GRAPH=$g LBMGPU_FUSED_MB=0 timeout 300 $B --config 1 --steps 100 > gpurun_out/r74/c1_perSweep_g$g.json 2> gpurun_out/r74/c1_g$g.err
  for k in aa-soa blk-push-soa blk-pull-soa; do
    LBMGPU_GRAPH=$g timeout 300 $B --config 1 --kernel $k --dims 96x96x96 --steps 100 > gpurun_out/r74/96_${k}_g$g.json 2> gpurun_out/r74/96_${k}_g$g.err
    LBMGPU_GRAPH=$g timeout 300 $B --config 1 --kernel $k --dims 128x128x128 --steps 100 > gpurun_out/r74/128_${k}_g$g.json 2> gpurun_out/r74/128_${k}_g$g.err
  done
  LBMGPU_GRAPH=$g timeout 300 $B > gpurun_out/r74/c5_g$g.json 2> gpurun_out/r74/c5_g$g.err
done

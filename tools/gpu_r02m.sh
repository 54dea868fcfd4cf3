#!/bin/bash
# Round 2m: parity of the staging tiles; ncu --set full of the list AoS odd tile (cfg 2)
TAG=${1:-r02m}
mkdir -p gpurun_out
[ -n "$SKIP_TESTS" ] || timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staging_tiles or guard_zones or edge_shapes" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
CMD="python bench.py --config 2 --kernel list-aa-aos --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
LBMGPU_LTILE=1 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
LBMGPU_LTILE=1 ncu --set full --clock-control none --import-source on -k regex:k_list_aa_odd_aos_tile -s 1 -c 1 -o gpurun_out/${TAG}_ltile $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?

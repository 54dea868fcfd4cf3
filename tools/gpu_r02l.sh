#!/bin/bash
# Round 2l: list-aa-aos staging tiles -- parity, then shapes on cfg 2 / cfg 4 (TAG from $1)
TAG=${1:-r02l}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staging_tiles or guard_zones or edge_shapes" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
for cfg in 2 4; do
for sh in ${SHAPES:-0 1 2 3 4 5}; do
  LBMGPU_LTILE=$sh timeout 300 python bench.py --config $cfg --kernel list-aa-aos --no-e2e --no-cpu-baseline --no-micro 2>gpurun_out/${TAG}_err_$cfg_$sh.txt | tail -1 > gpurun_out/${TAG}_cfg${cfg}_t$sh.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg${cfg}_t$sh.json'));print('cfg$cfg shape $sh', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
done

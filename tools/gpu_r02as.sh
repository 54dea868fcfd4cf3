#!/bin/bash
# Round 2as: persistent list-aa-aos staging tiles, second-CTA stagger sweep
TAG=${1:-r02as}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staging_tiles" 2>&1 | tail -1
for st in ${STAGGERS:-0 2000 4000 8000}; do
for cfg in 2 4; do
  LBMGPU_LTILE_STAGGER=$st timeout 300 python bench.py --config $cfg --kernel list-aa-aos --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg${cfg}_st$st.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg${cfg}_st$st.json'));print('cfg$cfg stagger $st', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

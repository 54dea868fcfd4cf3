#!/bin/bash
# Round 2z: list-aa-aos tile kernel, L2 prefetch distance sweep (TAG from $1)
TAG=${1:-r02z}
mkdir -p gpurun_out
for cfg in 2 4; do
for pf in ${PFS:-0 1 2 3 4 6}; do
  LBMGPU_LTILE=${SHAPE:-1} LBMGPU_LTILE_PF=$pf timeout 300 python bench.py --config $cfg --kernel list-aa-aos --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg${cfg}_pf$pf.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg${cfg}_pf$pf.json'));print('cfg$cfg pf $pf', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
done

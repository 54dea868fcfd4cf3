#!/bin/bash
# Round 2ap: EXPERIMENT two nodes per thread in the SoA AA sweeps (cfg 5)
TAG=${1:-r02ap}
mkdir -p gpurun_out
for x2 in 0 2 3 0; do
  LBMGPU_AA_X2=$x2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_x2$x2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_x2$x2.json').read().strip().splitlines()[-1]);print('x2 $x2', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done

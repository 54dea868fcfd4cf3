#!/bin/bash
TAG=r02f
mkdir -p gpurun_out
for t in 44 42 24; do
for k in aa-aos blk-push-aos; do
  LBMGPU_AOS_TILE=$t timeout 300 python bench.py --config 5 --kernel $k --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg5_${k}_t$t.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg5_${k}_t$t.json'));print('$k t$t', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
done
for k in aa-aos blk-push-aos blk-pull-aos; do
  timeout 300 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg1_${k}.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg1_${k}.json'));print('cfg1 $k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
timeout 600 python -m pytest tests/test_microbench.py -q > gpurun_out/${TAG}_micro.log 2>&1; tail -2 gpurun_out/${TAG}_micro.log

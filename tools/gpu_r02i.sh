#!/bin/bash
TAG=r02i
mkdir -p gpurun_out
for co in -1 50 33 20; do
for k in list-push-aos list-aa-aos; do
  LBMGPU_CARVEOUT=$co timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg2_${k}_co$co.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg2_${k}_co$co.json'));print('$k co$co', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
done
( time timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err ) 2> gpurun_out/${TAG}_ref.time; echo ref rc=$?
tail -1 gpurun_out/${TAG}_ref.json; cat gpurun_out/${TAG}_ref.time; free -g | head -2

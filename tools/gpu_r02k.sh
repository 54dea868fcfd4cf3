#!/bin/bash
# Round 2k: sanity of the rebuilt tree (smoke, default bench, AoS AA names)
TAG=r02k
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; tail -c 600 gpurun_out/${TAG}_bench.json
for k in list-aa-aos; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg2_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done

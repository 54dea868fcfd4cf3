#!/bin/bash
TAG=r02g
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
grep -E 'FAIL|Error' gpurun_out/${TAG}_pytest.log | head -10
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
for k in list-push-aos list-pull-aos list-aa-aos; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg2_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
timeout 600 python bench.py --virtual-parts 8 --steps 10 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg5_vp8.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg5_vp8.json'));print('vp8', round(d['value']), d.get('overlap'))"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print('bench', round(d['value']), d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline'])"

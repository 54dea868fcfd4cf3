#!/bin/bash
TAG=r02h
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle_steppers or aos or golden or fingerprint" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_pytest.log
for k in list-push-aos list-pull-aos; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg2_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
timeout 300 python bench.py --config 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg3.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg3.json'));print('cfg3', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
timeout 300 python bench.py --config 5 --kernel blk-pull-soa --steps 10 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg5_pull.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg5_pull.json'));print('cfg5 pull', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
/usr/bin/time -v timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
tail -1 gpurun_out/${TAG}_ref.json; grep -E 'Elapsed|Maximum resident' gpurun_out/${TAG}_ref.err

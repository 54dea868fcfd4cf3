#!/bin/bash
# Round 2a: GPU suite after the pruning + AoS push in pull order; AA launch-bound sweep; AoS names
TAG=r02a
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
for mb in 3 4 5 6; do
  LBMGPU_AA_MINB=$mb timeout 300 python bench.py --config 5 --steps 10 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg5_minb$mb.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg5_minb$mb.json'));print('minb $mb', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done
for k in blk-push-aos blk-pull-aos aa-aos blk-push-soa; do
  timeout 300 python bench.py --config 5 --kernel $k --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg5_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
for k in list-aa-aos list-push-aos list-pull-aos; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg2_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
timeout 300 python bench.py --config 1 --kernel blk-push-aos --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg1_blk-push-aos.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg1_blk-push-aos.json'));print('cfg1 push-aos', round(d['value']))"

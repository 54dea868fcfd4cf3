#!/bin/bash
TAG=r02e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "aos or zslab or node_range or list_parts" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -m pytest tests/test_dropin.py -q -x > gpurun_out/${TAG}_dropin.log 2>&1; echo dropin rc=$?; tail -2 gpurun_out/${TAG}_dropin.log
timeout 300 python bench.py --config 5 --kernel aa-aos --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_aa-aos.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg5_aa-aos.json'));print('aa-aos', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
LBMGPU_FUSED_MB=0 timeout 300 python bench.py --config 1 --kernel aa-aos --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg1_aa-aos_mb0.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg1_aa-aos_mb0.json'));print('cfg1 aa-aos mb0', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
CMD="python bench.py --config 5 --kernel aa-aos --dims 256x128x128 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:aa_odd_aos -s 1 -c 1 -o gpurun_out/${TAG}_aa_odd_aos $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?

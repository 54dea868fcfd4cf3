#!/bin/bash
TAG=r02c
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "aos or structure_bitwise" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
grep -i 'passed\|failed\|error' gpurun_out/${TAG}_pytest.log | head -5
timeout 300 python bench.py --config 5 --kernel aa-aos --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_aa-aos.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg5_aa-aos.json'));print('aa-aos', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
LBMGPU_FUSED_MB=0 timeout 300 python bench.py --config 1 --kernel aa-aos --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg1_aa-aos_mb0.json
python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg1_aa-aos_mb0.json'));print('cfg1 aa-aos mb0', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"

#!/bin/bash
# Round 2an: pipelined job with / without programmatic dependent launches; default bench
TAG=${1:-r02an}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "run_job" 2>&1 | tail -1
for pdl in 1 0 1 0; do
  LBMGPU_JOB_PDL=$pdl timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-micro > gpurun_out/${TAG}_pdl$pdl.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_pdl$pdl.json').read().strip().splitlines()[-1]);print('pdl $pdl', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['seconds'],3), d['e2e']['pipelined'], {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done

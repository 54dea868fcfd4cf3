#!/bin/bash
# Round 2ad: pipelined job (lbmgpu_run) e2e on cfg 5, slab / chunk sweep with the job trace
# CASES="slabs:chunk[:chunk_out] ..." (chunks in slabs)
TAG=${1:-r02ad}
mkdir -p gpurun_out
for sc in ${CASES:-256:8 192:6 128:4}; do
  IFS=: read S K KO <<< "$sc"; KO=${KO:-32}
  LBMGPU_JOB_SLABS=$S LBMGPU_JOB_CHUNK=$K LBMGPU_JOB_CHUNK_OUT=$KO LBMGPU_JOB_TRACE=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-micro > gpurun_out/${TAG}_s${S}_k${K}_o${KO}.json 2> gpurun_out/${TAG}_s${S}_k${K}_o${KO}.err
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_s${S}_k${K}_o${KO}.json').read().strip().splitlines()[-1]);print('slabs $S chunk $K out $KO', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['seconds'],3), d['e2e']['pipelined'])"
  grep -A200 "T=200" gpurun_out/${TAG}_s${S}_k${K}_o${KO}.err | tail -n +2 | tail -80 | awk 'NR%8==1 || NR==0'
done

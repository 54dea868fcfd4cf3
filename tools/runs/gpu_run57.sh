#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b57.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/p57.log 2>&1; echo rc=$? >> gpurun_out/p57.log
for dims in 32x32x32 64x64x64; do for k in list-aa-soa list-pull-soa list-push-soa list-aa-aos; do
  timeout 300 python bench.py --config 5 --kernel $k --dims $dims --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$dims', '$k', round(d['value']), list(d['kernels'])[0])" >> gpurun_out/b57.txt
done; done

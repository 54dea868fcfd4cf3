#!/bin/bash
# decomposition overhead probe on one GPU: device-copy vs NCCL-self halos
mkdir -p gpurun_out; rm -f gpurun_out/b61.txt
for vp in 1 2 4 8; do for t in "" "--nccl-self"; do
  if [ $vp = 1 ] && [ -n "$t" ]; then continue; fi
  timeout 300 python bench.py --config 5 --virtual-parts $vp $t --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 aa', $vp, '$t', round(d['value']))" >> gpurun_out/b61.txt
  timeout 300 python bench.py --config 5 --kernel blk-pull-soa --virtual-parts $vp $t --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 pull', $vp, '$t', round(d['value']))" >> gpurun_out/b61.txt
  timeout 300 python bench.py --config 5 --kernel blk-push-soa --virtual-parts $vp $t --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 push', $vp, '$t', round(d['value']))" >> gpurun_out/b61.txt
  timeout 300 python bench.py --config 2 --virtual-parts $vp $t --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 list', $vp, '$t', round(d['value']))" >> gpurun_out/b61.txt
done; done

#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/b38.txt
for k in aa-aos blk-push-aos blk-pull-aos; do for band in 0 2 4 16; do
LBMGPU_AOS_BAND=$band timeout 300 python bench.py --config 5 --kernel $k --dims 1024x512x128 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', $band, round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})" >> gpurun_out/b38.txt
done; done

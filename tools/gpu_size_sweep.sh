#!/bin/bash
# MFLUP/s against lattice size (channel boxes), one GPU: where the fused
# L2-resident launch applies and where the HBM roofline takes over
mkdir -p gpurun_out; rm -f gpurun_out/size_sweep.txt
for dims in 32x32x32 64x64x64 96x96x96 128x128x128 256x128x128 256x256x256 512x256x256 1024x512x256 1024x512x512; do
  for k in aa-soa blk-push-soa list-aa-soa; do
    if [ "$k" = "list-aa-soa" ] && [ "$dims" = "1024x512x512" ]; then continue; fi
    timeout 300 python bench.py --config 5 --kernel $k --dims $dims --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$dims', '$k', d['n_fluid'], round(d['value']), round(d['step_roofline_frac'],3), list(d['kernels'])[0])" >> gpurun_out/size_sweep.txt
  done
done

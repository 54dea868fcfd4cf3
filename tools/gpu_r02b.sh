#!/bin/bash
# Round 2b: AoS AA odd step with the owned-slot write-back; cfg 1 AoS fused vs tiles; peer timeout test
TAG=r02b
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "aos or oracle_steppers or snapshot_out or guard" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -m pytest tests/test_peer_ipc.py -q -x > gpurun_out/${TAG}_peer.log 2>&1; echo peer rc=$?
tail -3 gpurun_out/${TAG}_peer.log
for k in aa-aos; do
  timeout 300 python bench.py --config 5 --kernel $k --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg5_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
for k in blk-push-aos blk-pull-aos aa-aos; do
  for mb in 96 0; do
  LBMGPU_FUSED_MB=$mb timeout 300 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_cfg1_${k}_mb$mb.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_cfg1_${k}_mb$mb.json'));print('cfg1 $k mb$mb', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
  done
done

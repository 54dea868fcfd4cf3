#!/bin/bash
# Round 2bj: AoS 3-D tiles with the inner fast path, compile-time owner masks and the 3-D grid:
# parity, then aa-aos / blk-pull-aos / blk-push-aos on the cfg-5 box and cfg 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_kernels_ref.py tests/test_acceptance.py tests/test_full_lattice_ref.py -m gpu -x -q -k "aos or tiles or golden or criterion_5 or criterion_8 or stepper or guard or edge" 2>&1 | tail -3
for by in 8 0 4 16; do for k in aa-aos blk-pull-aos; do
  LBMGPU_TILE_BY=$by timeout 300 python bench.py --config 5 --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r02bj_${k}_$by.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02bj_${k}_$by.json').read().strip().splitlines()[-1]);print('by $by $k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done
for k in blk-push-aos; do
  timeout 300 python bench.py --config 5 --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r02bj_${k}.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02bj_${k}.json').read().strip().splitlines()[-1]);print('$k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done
for k in aa-aos blk-pull-aos; do
  timeout 300 python bench.py --config 1 --kernel $k --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r02bj_c1_${k}.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02bj_c1_${k}.json').read().strip().splitlines()[-1]);print('cfg1 $k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done

#!/bin/bash
# Round 2bn: fused (L2-resident) launches with 32-bit element indices: parity, then cfg 1 and 64^3 names
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_kernels_ref.py tests/test_acceptance.py -m gpu -x -q -k "golden or oracle_steppers or fused or launch_shapes or criterion_8 or edge or baseline_config_fingerprint" 2>&1 | tail -3
for k in blk-push-soa blk-pull-soa aa-soa blk-push-aos; do for st in 20 100; do
  timeout 300 python bench.py --config 1 --kernel $k --steps $st --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r02bn_${k}_$st.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02bn_${k}_$st.json').read().strip().splitlines()[-1]);print('cfg1 $k steps $st', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

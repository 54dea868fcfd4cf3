#!/bin/bash
# RIA pattern ids of 16/32 bits: parity, then cfg 4 / cfg 2 with list-aa-ria-soa
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ria" > gpurun_out/r67_pytest.log 2>&1; echo rc=$? >> gpurun_out/r67_pytest.log
timeout 600 python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r67_cfg4_ria.json 2> gpurun_out/r67_cfg4_ria.err
LBMGPU_RIA_MODE=0 timeout 600 python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r67_cfg4_ria_runtable.json 2> gpurun_out/r67_cfg4_ria_runtable.err
timeout 600 python bench.py --config 2 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/r67_cfg2_ria.json 2> gpurun_out/r67_cfg2_ria.err

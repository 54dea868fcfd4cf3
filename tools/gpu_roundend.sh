#!/bin/bash
# What the driver runs at round end: gpu tests, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/re_pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/re_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/re_smoke.log
python bench.py --impl reference > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo ref rc=$? >> gpurun_out/re_ref.err
python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo bench rc=$? >> gpurun_out/re_bench.err

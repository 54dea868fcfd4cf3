mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab or golden_bitwise or port_oracle or custom" > gpurun_out/pytest_gpu8.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu8.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b8.json 2>&1; echo rc=$?
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b8b.json 2>&1; echo rc=$?

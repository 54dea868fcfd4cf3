mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab or golden_bitwise or port_oracle or custom or fixed_point or mass" > gpurun_out/pytest_gpu12.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu12.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b12.json 2>&1; echo rc=$?

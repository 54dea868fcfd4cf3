mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu14.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu14.log
python bench.py --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b14.json 2>&1; echo rc=$?

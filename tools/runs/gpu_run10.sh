mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab" > gpurun_out/pytest_gpu10.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu10.log

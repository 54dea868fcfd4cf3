mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu9.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu9.log
python bench.py --no-cpu-baseline > gpurun_out/b9.json 2>&1; echo rc=$?

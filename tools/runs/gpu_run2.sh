set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --dims 1024x512x64 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:full_aa -s 2 -c 2 -o gpurun_out/prof_aa $B > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_full.log

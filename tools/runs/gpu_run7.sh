mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu7.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu7.log
python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench rc=$?

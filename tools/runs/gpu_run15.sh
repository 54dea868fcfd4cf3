mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu15.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu15.log
for c in 2 4; do for p in 0 1; do
LBMGPU_LIST_ODD_PIPE=$p python bench.py --config $c --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b15_c${c}_p$p.json 2>&1; echo c=$c p=$p rc=$?
done; done
for c in 1 3 5; do python bench.py --config $c --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b15_c${c}.json 2>&1; echo c=$c rc=$?; done

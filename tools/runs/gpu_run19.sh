mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or ria or blocking or mass or port" > gpurun_out/pytest_gpu19.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu19.log
for m in 0 1; do for w in 1 2; do
LBMGPU_RIA_MODE=$m LBMGPU_LIST_PF_WAVES=$w python bench.py --config 2 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b19_ria_m${m}_w$w.json 2>&1
done; done
python bench.py --config 4 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b19_c4.json 2>&1
python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b19_c4ria.json 2>&1
python bench.py --config 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b19_c3.json 2>&1

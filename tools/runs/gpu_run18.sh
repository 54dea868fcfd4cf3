mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or ria or blocking or mass" > gpurun_out/pytest_gpu18.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu18.log
for w in 0 1 2 4; do
LBMGPU_LIST_PF_WAVES=$w python bench.py --config 2 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b18_c2_w$w.json 2>&1; echo w=$w rc=$?
LBMGPU_LIST_PF_WAVES=$w python bench.py --config 2 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b18_c2ria_w$w.json 2>&1
done
LBMGPU_RIA_MODE=0 python bench.py --config 2 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b18_c2ria_mode0.json 2>&1
python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b18_c4ria.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "baseline_config_fingerprint" --durations=5 > gpurun_out/pytest_gpu18b.log 2>&1; echo cfgtests rc=$?
tail -8 gpurun_out/pytest_gpu18b.log

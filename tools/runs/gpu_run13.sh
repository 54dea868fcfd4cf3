mkdir -p gpurun_out
LBMGPU_AA_PIPE=22 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab or golden_bitwise or custom or fixed_point" > gpurun_out/pytest_gpu13.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu13.log
for p in 0 22 21 31 41; do
LBMGPU_AA_PIPE=$p python bench.py --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b13_$p.json 2>&1; echo p=$p rc=$?
done

mkdir -p gpurun_out
for mb in 1 3 4; do
  LBMGPU_AA_MINB=$mb python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b5_mb$mb.json 2>&1; echo mb=$mb rc=$?
done
LBMGPU_AA_MINB=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab or golden_bitwise" > gpurun_out/pytest_gpu5.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_gpu5.log

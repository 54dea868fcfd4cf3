mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu3.log
for st in 0 3 4 5; do
  LBMGPU_AA_TMA_STAGES=$st python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b3_st$st.json 2>&1; echo st=$st rc=$?
done
LBMGPU_AA_TMA_STAGES=0 LBMGPU_AA_CS=1 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b3_cs.json 2>&1; echo cs rc=$?

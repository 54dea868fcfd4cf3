mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "zslab or golden_bitwise or port_oracle" > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu4.log
for st in 0 3 4 5 12; do
  LBMGPU_AA_TMA_STAGES=$st python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b4_st$st.json 2>&1; echo st=$st rc=$?
done

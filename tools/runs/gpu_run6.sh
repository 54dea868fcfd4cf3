mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.mem,clocks.max.mem,clocks.sm,temperature.gpu,power.draw --format=csv
for i in 1 2; do for mb in 1 3; do
  LBMGPU_AA_MINB=$mb python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b6_mb${mb}_$i.json 2>&1; echo mb=$mb rc=$?
done; done
nvidia-smi --query-gpu=clocks.mem,clocks.max.mem,clocks.sm,temperature.gpu,power.draw --format=csv

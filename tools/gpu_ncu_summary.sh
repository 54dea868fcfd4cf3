#!/bin/bash
# Regenerates the committed DRAM-traffic capture behind roofline.traffic:
# per-launch dram bytes of every BASELINE config's default kernel, stamped
# with the csrc content hash of the tree it ran (tools/ncu_summary.py build).
mkdir -p gpurun_out
python -c "import bench; print(bench.csrc_sha16())" > gpurun_out/ncu_csrc_sha16.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 5 2 3 4 1; do
  if [ $c = 1 ]; then A="--steps 20 --warmup 0"; else A="--steps 2 --warmup 1"; fi
  CMD="python bench.py --config $c $A --no-e2e --no-cpu-baseline --no-micro"
  $CMD > gpurun_out/ncu_plain_cfg$c.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_cfg$c.csv $CMD > gpurun_out/ncu_run_cfg$c.log 2>&1
  echo cfg$c ncu rc=$?
done

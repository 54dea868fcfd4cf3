#!/bin/bash
# ncu launch lists (time + DRAM bytes) for the list configs and the ria/pid and AoS kernels
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in "2 list-aa-soa" "3 list-pull-soa" "4 list-aa-soa" "2 list-aa-ria-soa" "4 list-aa-ria-soa" "1 blk-push-soa"; do
  set -- $spec
  B="python bench.py --config $1 --kernel $2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
  $B > gpurun_out/r01e_plain_$1_$2.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:"k_list|k_full_fused" -c 12 --csv --log-file gpurun_out/r01e_launches_$1_$2.csv $B > gpurun_out/r01e_ncu_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
done

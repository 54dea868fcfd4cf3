#!/bin/bash
# AA temporal blocking: does the pair's second touch hit L2? ncu DRAM bytes for small live windows
mkdir -p gpurun_out/r78
for tb in 16,2 32,1 8,4 64,1; do
  LBMGPU_AA_TB=$tb timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-micro --steps 4 --warmup 3 > gpurun_out/r78/c5_$tb.json 2> gpurun_out/r78/c5_$tb.err
  LBMGPU_AA_TB=$tb timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:aa_tb -c 1 --csv --log-file gpurun_out/r78/ncu_$tb.csv python bench.py --no-e2e --no-cpu-baseline --no-micro --steps 2 --warmup 3 > gpurun_out/r78/ncu_$tb.log 2>&1
done

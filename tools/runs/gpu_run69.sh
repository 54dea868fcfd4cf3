#!/bin/bash
# ncu --set full of the RIA odd step with 32-bit pattern ids (cfg 4) + launch list
mkdir -p gpurun_out
C="python bench.py --config 4 --kernel list-aa-ria-soa --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$C > gpurun_out/r69_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:odd_pid -s 2 -c 1 -o gpurun_out/r69_prof_pid32 $C > gpurun_out/r69_ncu.log 2>&1; echo rc=$? >> gpurun_out/r69_ncu.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/r69_launches.csv $C > gpurun_out/r69_ncu2.log 2>&1

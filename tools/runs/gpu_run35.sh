#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --kernel aa-aos --dims 1024x512x128 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/b35_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:k_full_aa -c 6 --csv \
    --log-file gpurun_out/b35_aos.csv $B > gpurun_out/b35_ncu.log 2>&1; echo rc=$?

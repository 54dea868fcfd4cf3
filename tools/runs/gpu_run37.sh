#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --kernel aa-aos --dims 1024x512x128 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
for band in 0 16 4; do
LBMGPU_AOS_BAND=$band $B > gpurun_out/b37_plain_$band.log 2>&1 && \
LBMGPU_AOS_BAND=$band ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_full_aa_odd -c 2 --csv \
    --log-file gpurun_out/b37_$band.csv $B > gpurun_out/b37_ncu_$band.log 2>&1; echo rc=$?
done

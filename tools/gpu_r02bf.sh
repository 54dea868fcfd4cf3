#!/bin/bash
# Round 2bf: ncu --set full of the direct AoS AA odd tile kernel, every lts / dram / l1tex metric
mkdir -p gpurun_out
CMD="python bench.py --config 5 --kernel aa-aos --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro --dims 1024x512x64"
$CMD > gpurun_out/r02bf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_full_aa_odd_aos_tile3d -s 1 -c 1 -o gpurun_out/r02bf_aa_aos $CMD > gpurun_out/r02bf_ncu.log 2>&1
echo ncu rc=$?
ncu -i gpurun_out/r02bf_aa_aos.ncu-rep --page raw --csv > gpurun_out/r02bf_aa_aos_raw.csv 2>/dev/null
ls -la gpurun_out/r02bf*

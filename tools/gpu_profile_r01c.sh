#!/bin/bash
# Round-1c evidence: headline bench line (cfg 5 with e2e + cpu baseline), all
# configs, cfg 5 launch list, full ncu of the AA pair (reduced z) and of the
# cfg-1 fused push launch.
TAG=r01c
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err; echo bench rc=$?
for c in 1 2 3 4; do python bench.py --config $c --no-micro > gpurun_out/${TAG}_bench_cfg$c.json 2> gpurun_out/${TAG}_bench_cfg$c.err; echo c$c rc=$?; done
python bench.py --config 2 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/${TAG}_bench_cfg2_ria.json 2>&1
python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/${TAG}_bench_cfg4_ria.json 2>&1
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/${TAG}_cfg5_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches rc=$?
S="python bench.py --dims 1024x512x64 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$S > gpurun_out/${TAG}_plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:full_aa -s 2 -c 2 -o gpurun_out/${TAG}_prof_aa $S \
    > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full rc=$?
C="python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-micro"
$C > gpurun_out/${TAG}_plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/${TAG}_prof_c1 $C \
    > gpurun_out/${TAG}_ncu_c1.log 2>&1; echo c1 rc=$?

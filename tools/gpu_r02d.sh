#!/bin/bash
TAG=r02d
mkdir -p gpurun_out
./integration/_build/dropin_check > gpurun_out/${TAG}_dropin.log 2>&1; echo dropin rc=$?
cat gpurun_out/${TAG}_dropin.log
CMD="python bench.py --config 5 --kernel aa-aos --dims 256x128x128 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:aa_odd_aos -s 1 -c 1 -o gpurun_out/${TAG}_aa_odd_aos $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?

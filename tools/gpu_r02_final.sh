#!/bin/bash
# Round-2 numbers on the final code: every BASELINE config's bench line (e2e, CPU
# baseline), every other name on the BASELINE geometries, then the ncu DRAM
# traffic capture behind roofline.traffic (tools/gpu_ncu_summary.sh).
TAG=${1:-r02z}
mkdir -p gpurun_out
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --no-micro > gpurun_out/${TAG}_bench_cfg$c.json 2> gpurun_out/${TAG}_bench_cfg$c.err; echo cfg$c rc=$?
done
for k in list-aa-ria-soa list-aa-pv-soa list-aa-aos list-pull-aos list-push-soa list-push-aos list-pull-split-nt-2s-soa list-pull-split-nt-1s-soa; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json; done
for k in list-aa-ria-soa list-aa-aos; do
  timeout 300 python bench.py --config 4 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg4_$k.json; done
for k in aa-vec-soa aa-aos blk-push-soa blk-pull-soa blk-push-aos blk-pull-aos; do
  timeout 300 python bench.py --config 5 --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_$k.json; done
echo names done
[ -n "$NO_NCU" ] || bash tools/gpu_ncu_summary.sh

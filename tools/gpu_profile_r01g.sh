#!/bin/bash
# Round-1g bench lines after the cooperative-groups grid sync, halo tiles and the fused list launch
TAG=r01g
mkdir -p gpurun_out
python bench.py --config 1 --no-micro > gpurun_out/${TAG}_bench_cfg1.json 2> gpurun_out/${TAG}_bench_cfg1.err; echo c1 rc=$?
for k in list-aa-ria-soa list-aa-pv-soa list-aa-aos list-pull-aos list-push-soa list-push-aos list-pull-split-nt-2s-soa list-pull-split-nt-1s-soa; do
  python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json; done
python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg4_list-aa-ria-soa.json
for k in aa-vec-soa aa-aos blk-push-soa blk-pull-soa blk-push-aos blk-pull-aos; do
  python bench.py --config 5 --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_$k.json; done

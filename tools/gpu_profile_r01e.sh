#!/bin/bash
# Round-1e bench lines: every config (with e2e + CPU baseline) and the other names on the BASELINE geometries
TAG=r01e
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err; echo c5 rc=$?
for c in 1 2 3 4; do python bench.py --config $c --no-micro > gpurun_out/${TAG}_bench_cfg$c.json 2> gpurun_out/${TAG}_bench_cfg$c.err; echo c$c rc=$?; done
for k in list-aa-ria-soa list-aa-pv-soa list-aa-aos list-pull-aos list-push-soa list-push-aos list-pull-split-nt-2s-soa; do
  python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json; done
python bench.py --config 4 --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg4_list-aa-ria-soa.json
for k in aa-vec-soa aa-aos blk-push-soa blk-pull-soa blk-push-aos blk-pull-aos; do
  python bench.py --config 5 --kernel $k --steps 6 --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg5_$k.json; done

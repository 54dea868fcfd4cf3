#!/bin/bash
# final per-config bench lines of round 1h (every BASELINE config, full contract line)
mkdir -p gpurun_out/r80
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/r80/cfg$c.json 2> gpurun_out/r80/cfg$c.err
done
timeout 900 python bench.py > gpurun_out/r80/cfg5.json 2> gpurun_out/r80/cfg5.err

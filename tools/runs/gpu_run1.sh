set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo rc=$?
tail -3 gpurun_out/bench_cfg5.err
for c in 1 2 3 4; do python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2>gpurun_out/bench_cfg$c.err; echo cfg$c rc=$?; done
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu rc=$?

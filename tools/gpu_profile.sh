# Round profile capture: bench line, ncu launch list (cfg 5) and one full ncu
# capture of the AA pair on a reduced-z cfg-5 box.  Usage: bash tools/gpu_profile.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches rc=$?
S="python bench.py --dims 1024x512x64 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$S > gpurun_out/${TAG}_plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:full_aa -s 2 -c 2 -o gpurun_out/${TAG}_prof_aa $S \
    > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full rc=$?

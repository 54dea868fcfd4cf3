mkdir -p gpurun_out
for vp in 1 2 4 8; do
python bench.py --virtual-parts $vp --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b21_c5_vp$vp.json 2>&1; echo vp=$vp rc=$?
done
for vp in 1 4 8; do
python bench.py --config 2 --virtual-parts $vp --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b21_c2_vp$vp.json 2>&1; echo c2 vp=$vp rc=$?
done

# AoS direct names on the cfg-5 box and cfg 1
for k in ${KS:-aa-aos blk-pull-aos blk-push-aos}; do for c in 5 1; do
  timeout 300 python bench.py --config $c --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/aosb_${k}_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/aosb_${k}_$c.json').read().strip().splitlines()[-1]);print('cfg$c $k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

# list AoS names on cfg 2 / cfg 4
for k in ${KS:-list-pull-aos list-push-aos list-aa-aos}; do for c in ${CFGS:-2 4}; do
  timeout 300 python bench.py --config $c --kernel $k --no-e2e --no-cpu-baseline --no-micro > gpurun_out/laosb_${k}_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/laosb_${k}_$c.json').read().strip().splitlines()[-1]);print('cfg$c $k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

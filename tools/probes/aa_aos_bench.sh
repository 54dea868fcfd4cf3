for c in 5 1; do
  timeout 300 python bench.py --config $c --kernel aa-aos --steps 10 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/aab_$c.json 2> gpurun_out/aab_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/aab_$c.json').read().strip().splitlines()[-1]);print('cfg$c aa-aos', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done

for by in ${BYS:-0 2 4 8 16}; do for k in aa-aos blk-pull-aos; do
  LBMGPU_TILE_BY=$by timeout 300 python bench.py --config 5 --kernel $k --steps 10 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/tby_${k}_$by.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/tby_${k}_$by.json').read().strip().splitlines()[-1]);print('by $by $k', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

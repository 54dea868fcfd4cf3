for pp in 1 0 1 0; do for st in 20 50; do
  LBMGPU_PUSH_AS_PULL=$pp timeout 300 python bench.py --config 1 --steps $st --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/c1pp_${pp}_$st.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c1pp_${pp}_$st.json').read().strip().splitlines()[-1]);print('as_pull $pp steps $st', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

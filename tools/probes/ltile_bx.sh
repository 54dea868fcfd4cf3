for bx in ${BXS:-0 2 4 8 16}; do for c in 2 4; do
  LBMGPU_LTILE_BX=$bx timeout 300 python bench.py --config $c --kernel list-aa-aos --no-e2e --no-cpu-baseline --no-micro > gpurun_out/lbx_${c}_$bx.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/lbx_${c}_$bx.json').read().strip().splitlines()[-1]);print('bx $bx cfg$c', round(d['value']), {k:round(v['achieved_GBps']) for k,v in d['kernels'].items()})"
done; done

mkdir -p gpurun_out
python -c "
import paper_1711_11468_b200 as L
for k in ['copy','copy-19','copy-19-nt-sl','update-19']:
    print(k, round(L.lbmgpu.microbench(k, 8<<30, 5),1))
for k in ['copy','update-19']:
    print(k, '32GB', round(L.lbmgpu.microbench(k, 32<<30, 5),1))
" > gpurun_out/micro11.log 2>&1; echo micro rc=$?
cat gpurun_out/micro11.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/b11.json 2>&1; echo rc=$?

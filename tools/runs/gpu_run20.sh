mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu20.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu20.log
for i in 1 2; do python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b20_c1_$i.json 2>&1; done
LBMGPU_FUSED_MB=0 python bench.py --config 1 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b20_c1_nofuse.json 2>&1
python bench.py --config 1 --steps 50 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b20_c1_50.json 2>&1
python -c "
import time, paper_1711_11468_b200 as L
for n in ['aa-soa','list-aa-soa','blk-push-soa']:
    t=time.time(); r=L.verify_kernel(n, L.PoiseuilleCase(8,8,34,1e-6,L.TrtParams.from_tau(0.9)), check_interval=500, rel_tol=3e-8, max_steps=100000); print(n, r['steps'], r['passed'], round(time.time()-t,2),'s')
" > gpurun_out/verify_time20.log 2>&1; cat gpurun_out/verify_time20.log

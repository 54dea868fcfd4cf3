#!/bin/bash
# AA temporal blocking prototype: parity, then cfg 5 with several (W, G), ncu DRAM bytes of one
mkdir -p gpurun_out/r77
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "temporal" > gpurun_out/r77/pytest.log 2>&1; echo rc=$? >> gpurun_out/r77/pytest.log
grep -q "rc=0" gpurun_out/r77/pytest.log || exit 0
B="python bench.py --no-e2e --no-cpu-baseline --no-micro --steps 4 --warmup 3"
for tb in 64,4 32,8 128,2 64,2 128,4 256,2 512,1; do
  LBMGPU_AA_TB=$tb timeout 300 $B > gpurun_out/r77/c5_$tb.json 2> gpurun_out/r77/c5_$tb.err
done
LBMGPU_AA_TB=128,2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:aa_tb -c 1 --csv --log-file gpurun_out/r77/ncu_128_2.csv python bench.py --no-e2e --no-cpu-baseline --no-micro --steps 2 --warmup 3 > gpurun_out/r77/ncu.log 2>&1

#!/bin/bash
# Round 2j: full GPU suite, parity fuzzing, AoS list names, then the ncu captures
TAG=r02j
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python tools/fuzz_parity.py 400 31000 > gpurun_out/${TAG}_fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/${TAG}_fuzz.log
FUZZ_BIG=1 timeout 900 python tools/fuzz_parity.py 100 32000 > gpurun_out/${TAG}_fuzz_big.log 2>&1; echo fuzzbig rc=$?; tail -1 gpurun_out/${TAG}_fuzz_big.log
for k in list-push-aos list-pull-aos list-aa-aos; do
  timeout 300 python bench.py --config 2 --kernel $k --no-e2e --no-cpu-baseline --no-micro 2>/dev/null | tail -1 > gpurun_out/${TAG}_names_cfg2_$k.json
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_names_cfg2_$k.json'));print('$k', round(d['value']), {k:(round(v['achieved_GBps']),round(v['share'],3)) for k,v in d['kernels'].items()})"
done
bash tools/gpu_ncu_summary.sh
CMD="python bench.py --config 5 --dims 1024x512x64 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-micro"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_full_aa -s 2 -c 2 -o gpurun_out/${TAG}_aa_soa $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu rc=$?

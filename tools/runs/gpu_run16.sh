mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or ria or blocking or mass or fixed" > gpurun_out/pytest_gpu16.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu16.log
for c in 2 4; do
python bench.py --config $c --kernel list-aa-ria-soa --no-e2e --no-cpu-baseline --no-micro > gpurun_out/b16_c${c}_ria.json 2>&1; echo c=$c rc=$?
done
python -c "
import paper_1711_11468_b200 as L
for spec in [L.GeometrySpec('channel',256,256,256), L.GeometrySpec('blocks',400,400,400,8,8)]:
    k=L.make_kernel(L.make_descriptor('list-aa-ria-soa'), spec)
    print(spec.kind, k.n_fluid(), k.ria_stats(), k.vector_fraction())
" > gpurun_out/ria_stats16.log 2>&1; cat gpurun_out/ria_stats16.log

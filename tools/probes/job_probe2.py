"""Store-leg rate of the pipelined job vs chunk width and buffer aliasing."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1711_11468_b200 as lbm
k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 1024, 512, 512))
n = k.n_fluid() * 19
a = lbm.PinnedBuffer(n); a.array[:] = 0.05
b = lbm.PinnedBuffer(n); b.array[:] = 0.0
P, F = lbm.TrtParams(), lbm.BodyForce((1e-5, 0, 0))
for chunk in ("16", "32", "40"):
    os.environ["LBMGPU_JOB_CHUNK"] = chunk
    for inplace in (True, False):
        k.run(a.array, P, F, 2, out=a.array if inplace else b.array)
        k.synchronize(); t = time.perf_counter()
        k.run(a.array, P, F, 2, out=a.array if inplace else b.array)
        print(f"chunk {chunk} in-place {inplace}: {time.perf_counter() - t:.3f} s", flush=True)

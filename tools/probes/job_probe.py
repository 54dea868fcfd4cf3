"""Pipelined job on the cfg-5 box with few steps: the transfer legs alone
(LBMGPU_JOB_TRACE timeline on stderr), plus the plain load_state / snapshot
rates in the same process for comparison."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1711_11468_b200 as lbm
os.environ["LBMGPU_JOB_TRACE"] = "1"
k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 1024, 512, 512))
n = k.n_fluid() * 19
buf = lbm.PinnedBuffer(n)
buf.array[:] = 0.05
P, F = lbm.TrtParams(), lbm.BodyForce((1e-5, 0, 0))
for steps in (2, 2, 20):
    k.synchronize(); t = time.perf_counter()
    _, piped = k.run(buf.array, P, F, steps, out=buf.array)
    print(f"run steps={steps} pipelined={piped}: {time.perf_counter() - t:.3f} s", flush=True)
t = time.perf_counter(); k.load_state(buf.array); k.synchronize(); tl = time.perf_counter() - t
t = time.perf_counter(); k.snapshot(buf.array); k.synchronize(); ts = time.perf_counter() - t
print(f"plain load_state {n * 8 / tl / 1e9:.1f} GB/s, snapshot {n * 8 / ts / 1e9:.1f} GB/s", flush=True)

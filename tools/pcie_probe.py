import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1711_11468_b200 as lbm
x = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(4 << 30, dtype=torch.uint8, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); h2d=4/(time.perf_counter()-t)*1.073741824
    torch.cuda.synchronize(); t=time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); d2h=4/(time.perf_counter()-t)*1.073741824
print(f"raw pinned h2d {h2d:.1f} GB/s d2h {d2h:.1f} GB/s", flush=True)
del x, d
k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 1024, 512, 128))
buf = lbm.PinnedBuffer(k.n_fluid() * 19)
arr = buf.array
arr[:] = 0.05
for _ in range(2):
    k.synchronize(); t=time.perf_counter(); k.load_state(arr); k.synchronize(); tl=time.perf_counter()-t
    t=time.perf_counter(); k.snapshot(arr); k.synchronize(); ts=time.perf_counter()-t
nb = k.n_fluid()*19*8/1e9
print(f"load_state {nb/tl:.1f} GB/s snapshot {nb/ts:.1f} GB/s ({nb:.1f} GB)", flush=True)

"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel name on a tiny blocks box, the z-slab split, RIA, the
TMA-staged and cp.async-pipelined AA variants, snapshot/load and one short
verification.  Run as:  compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1711_11468_b200 as lbm  # noqa: E402

P, F = lbm.TrtParams.from_tau(0.9), lbm.BodyForce((1e-5, 2e-6, -3e-6))
spec = lbm.GeometrySpec("blocks", 12, 10, 10)
for name in lbm.kernel_names():
    k = lbm.make_kernel(lbm.make_descriptor(name, blk=2 if "list" in name else 0), spec)
    k.load_perturbed(1)
    k.advance(P, F, 4)
    s = k.snapshot()
    k.load_state(s)
    k.total_mass()
    if name.startswith("list-"):
        k.export_structure()
for parts in (2, 3):
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 16, 12, 24),
                        dist={"virtual_parts": parts})
    k.load_perturbed(2)
    k.advance(P, F, 4)
    k.snapshot_local()
# AoS 3-D halo tiles (nx % 16, ny / nz % 4)
for name in ("blk-push-aos", "blk-pull-aos", "aa-aos"):
    k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec("channel", 32, 12, 8))
    k.load_perturbed(3)
    k.advance(P, F, 4)
r = lbm.verify_kernel("aa-soa", lbm.PoiseuilleCase(4, 4, 10, 1e-6, P), check_interval=50,
                      max_steps=200)
print("sanitize cases done")

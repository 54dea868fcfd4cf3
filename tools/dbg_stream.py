import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_11468_b200 as lbm
from oracle.oracle import Port
port = Port()
P = lbm.TrtParams.from_tau(0.9); F = lbm.BodyForce((1e-5, 2e-6, -3e-6))
os.environ["LBMGPU_FUSED_MB"] = "0"
for guard in ("0", "1"):
    os.environ["LBMGPU_GUARD"] = guard
    for shape in sys.argv[1:]:
        os.environ["LBMGPU_LTILE"] = shape
        for kind, dims in [("channel", (32, 12, 8)), ("channel", (64, 64, 64)), ("blocks", (40, 36, 44))]:
            _, _, nf = port.geometry(kind, *dims)
            init = port.perturbed(nf, 5)
            try:
                k = lbm.make_kernel(lbm.make_descriptor("list-aa-aos"), lbm.GeometrySpec(kind, *dims))
                k.load_state(init)
                k.advance(P, F, 4)
                got = k.snapshot()
                exp, _ = port.run("half", kind, *dims, 4, P.omega_plus, g=(1e-5, 2e-6, -3e-6), init=init)
                print(guard, shape, kind, dims, "equal" if np.array_equal(got, exp) else "DIFF", flush=True)
            except Exception as e:
                print(guard, shape, kind, dims, "ERROR", e, flush=True)
                sys.exit(1)

"""Seeded random parity fuzzing on the GPU against the oracle's textbook
steppers (test infrastructure; the 32-case subset runs in
tests/test_gpu_parity.py::test_randomized_against_oracle).

    [FUZZ_BIG=1] python tools/fuzz_parity.py [cases] [seed0]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1711_11468_b200 as lbm  # noqa: E402
from oracle.oracle import Port  # noqa: E402

port = Port()
names = lbm.kernel_names()
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 500
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
bad = 0
jobs = piped_jobs = 0
for case in range(cases):
    rng = np.random.default_rng(seed0 + case)
    # a fifth of the cases: a pipelined job (direct SoA AA, column-uniform
    # geometry, per-sweep launches) through lbmgpu_run
    piped_case = rng.random() < 0.2
    while True:
        kind = str(rng.choice(["channel", "slit"] if piped_case else
                              ["channel", "slit", "pipe", "blocks"]))
        big = os.environ.get("FUZZ_BIG") == "1"  # boxes up to 128 x 48 x 48
        nx = (int(rng.choice([16, 32, 48, 64, 128] if big else [16, 32, 48, 64]))
              if rng.random() < 0.5 else int(rng.integers(1, 130 if big else 40)))
        ny, nz = int(rng.integers(3, 49 if big else 26)), int(rng.integers(3, 49 if big else 26))
        if rng.random() < 0.3:  # AoS 3-D halo-tile shapes (ny, nz multiples of 4)
            ny, nz = 4 * ((ny + 3) // 4), 4 * ((nz + 3) // 4)
        block, spacing = int(rng.integers(1, 5)), int(rng.integers(0, 4))
        try:
            _, _, nf = port.geometry(kind, nx, ny, nz, block, spacing)
        except ValueError:
            continue
        if nf > 0:
            break
    name = str(rng.choice(["aa-soa", "aa-vec-soa"] if piped_case else names))
    if name in ("aa-aos", "blk-pull-aos", "blk-push-aos") and rng.random() < 0.6:
        # direct AoS tiles with interior tiles (fixed-offset fast path) beside
        # the surface ones: three or more x tiles, three or more y / z tiles
        while True:
            kind = str(rng.choice(["channel", "slit", "pipe", "blocks"]))
            nx, ny, nz = (int(rng.choice([48, 64, 80])), 4 * int(rng.integers(3, 7)),
                          4 * int(rng.integers(3, 7)))
            try:
                _, _, nf = port.geometry(kind, nx, ny, nz, block, spacing)
            except ValueError:
                continue
            if nf > 0:
                break
        os.environ["LBMGPU_TILE_BY"] = str(rng.choice(["8", "0", "2", "3", "4"]))
    blk = int(rng.integers(0, 5)) if name.startswith("list-") else 0
    tau = float(rng.uniform(0.52, 1.95))
    g = tuple(float(v) for v in rng.uniform(-3e-5, 3e-5, 3))
    steps = int(rng.integers(1, 6)) * 2 if "aa" in name.split("-") else int(rng.integers(1, 11))
    os.environ["LBMGPU_FUSED_MB"] = "0" if piped_case else str(rng.choice(["96", "0"]))
    parts = 1 if piped_case else int(rng.choice([1, 1, 2, 3]))
    dist = None
    if parts > 1 and nz >= parts and (name in ("aa-soa", "aa-vec-soa", "blk-push-soa", "blk-pull-soa")
                                      or (name in ("list-aa-soa", "list-aa-aos") and blk == 0)):
        dist = {"virtual_parts": parts}
        if not name.startswith("list") and rng.random() < 0.5:
            dist["transport"] = "peer"  # boundary odd sweeps in the neighbour slab, epoch flags
    os.environ["LBMGPU_RIA_MODE"] = str(rng.choice(["-1", "0", "1", "2"]))  # ria / pv names
    os.environ["LBMGPU_LTILE"] = str(rng.choice(["1", "2", "5"]))  # list-aa-aos staging tiles
    # one job through lbmgpu_run (pipelined for direct SoA AA, column-uniform
    # geometries, page-locked buffers) instead of load_state / advance /
    # snapshot, with random slab / chunk widths
    job = dist is None and (piped_case or rng.random() < 0.35)
    os.environ["LBMGPU_JOB_SLABS"] = str(int(rng.integers(1, 600)))
    os.environ["LBMGPU_JOB_CHUNK"] = str(int(rng.integers(1, 40)))
    os.environ["LBMGPU_JOB_CHUNK_OUT"] = str(int(rng.integers(1, 40)))
    init = port.perturbed(nf, seed0 + case)
    fam = "half" if name.startswith("list-") else "full"
    params = lbm.TrtParams.from_tau(tau)
    expect, _ = port.run(fam, kind, nx, ny, nz, steps, params.omega_plus, g=g, init=init,
                         block=block, spacing=spacing)
    try:
        k = lbm.make_kernel(lbm.make_descriptor(name, blk=blk),
                            lbm.GeometrySpec(kind, nx, ny, nz, block, spacing), dist=dist)
        if job:
            bin_, bout = lbm.PinnedBuffer(nf * 19), lbm.PinnedBuffer(nf * 19)
            bin_.array[:] = init
            out, piped = k.run(bin_.array, params, lbm.BodyForce(g), steps, out=bout.array)
            ok = np.array_equal(out, expect)
            jobs += 1
            piped_jobs += int(piped)
            bin_.free()
            bout.free()
        else:
            k.load_state(init)
            k.advance(params, lbm.BodyForce(g), steps)
            ok = np.array_equal(k.snapshot(), expect)
        del k
    except lbm.ConfigError as e:  # e.g. more parts than fluid nodes
        print("config", case, name, kind, (nx, ny, nz), dist, e)
        continue
    if not ok:
        bad += 1
        print("MISMATCH", case, name, kind, (nx, ny, nz), block, spacing, blk, tau, steps,
              os.environ["LBMGPU_FUSED_MB"], os.environ["LBMGPU_RIA_MODE"],
              os.environ["LBMGPU_LTILE"], dist, "job" if job else "",
              os.environ["LBMGPU_JOB_SLABS"], os.environ["LBMGPU_JOB_CHUNK"],
              os.environ["LBMGPU_JOB_CHUNK_OUT"], flush=True)
print(f"{cases} cases ({jobs} through lbmgpu_run, {piped_jobs} pipelined), {bad} mismatches",
      flush=True)
sys.exit(1 if bad else 0)

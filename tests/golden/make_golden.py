"""Generates the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/liblbm_ref.so, built by `make -C oracle` from
/root/reference/proj/src) through its own API: make_kernel(make_descriptor),
load_state / advance / snapshot / total_mass / state_fingerprint,
build_structure, padding_offsets.  Run in this container (the GPU box has no
/root/reference):

    python tests/golden/make_golden.py small      # seconds
    python tests/golden/make_golden.py edge       # seconds
    python tests/golden/make_golden.py configs    # BASELINE configs 1-4, ~25 min
    python tests/golden/make_golden.py nodes      # node-list FNVs of cfgs 2-4, ~1 min
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Ref  # noqa: E402

TAU, G_TEST = 0.9, (1e-5, 2e-6, -3e-6)  # tests/test_kernels.cpp:14-15
BASE_G = (1e-5, 0.0, 0.0)               # BASELINE.json physics: omega+=1, Lambda=3/16


def small(ref: Ref):
    """Every kernel on the reference's own kernel-test geometry (blocks
    12x10x10, tests/test_kernels.cpp:17-19) and two more shapes, perturbed
    init (seed 1234), 8 steps, plus family snapshots as .npz."""
    out = {"cases": []}
    arrays = {}
    cases = [("blocks", (12, 10, 10), dict(block=4, spacing=4)),
             ("channel", (16, 12, 10), {}),
             ("pipe", (9, 12, 13), {}),
             ("slit", (6, 5, 9), {})]
    for kind, dims, kw in cases:
        for name in ref.kernel_names():
            k = ref.kernel(name, kind, *dims, threads=2, **kw)
            init = ref.perturbed(k.n_fluid, 1234)
            k.load_state(init)
            k.advance(1.0 / TAU, 3.0 / 16.0, G_TEST, 8)
            snap = k.snapshot()
            fam = "half" if name.startswith("list-") else "full"
            key = f"{kind}_{'x'.join(map(str, dims))}_{fam}"
            if key not in arrays:
                arrays[key] = snap
            else:
                assert np.array_equal(arrays[key], snap), (key, name)
            out["cases"].append({"kernel": name, "kind": kind, "dims": dims, **kw,
                                 "seed": 1234, "steps": 8, "tau": TAU, "g": G_TEST,
                                 "n_fluid": k.n_fluid, "fingerprint": f"{ref.fingerprint(snap):016x}",
                                 "mass": k.total_mass(), "snapshot_key": key})
    # structures: nodes/adjacency fingerprints for blk, padding, orientation, layout
    out["structures"] = []
    for kind, dims, kw in cases[:3]:
        for layout in ("soa", "aos"):
            for blk in (0, 2, 3):
                for pad in ("none", "auto", "thrash"):
                    if layout == "aos" and pad != "none":
                        continue
                    for scatter in (False, True):
                        s = ref.structure(kind, *dims, layout=layout, blk=blk, padding=pad,
                                          scatter=scatter, **kw)
                        out["structures"].append({
                            "kind": kind, "dims": dims, **kw, "layout": layout, "blk": blk,
                            "padding": pad, "scatter": scatter, "n_fluid": s["n_fluid"],
                            "starts": [int(v) for v in s["starts"]], "total_slots": s["total_slots"],
                            "adj_fnv": f"{ref.fingerprint_u32(s['adj']):016x}",
                            "nodes_fnv": f"{ref.fingerprint_u32(s['nodes'].astype(np.uint32)):016x}"})
    # padding KATs at the BASELINE list sizes
    out["padding"] = []
    for n in (16516096, 25956352, 25394208, 56000000, 1136):
        for mode in ("none", "auto", "thrash"):
            st, tot = ref.padding_offsets(n, mode)
            out["padding"].append({"n_fluid": n, "mode": mode, "starts": [int(v) for v in st],
                                   "total": tot})
    # RIA run statistics (build_ria / vectorizable_fraction)
    out["ria"] = []
    for kind, dims, kw, blk in [("channel", (20, 10, 10), {}, 0), ("channel", (20, 10, 10), {}, 2),
                                ("blocks", (12, 10, 10), dict(block=4, spacing=4), 0)]:
        runs, v = ref.ria(kind, *dims, blk=blk, vector_width=4, **kw)
        out["ria"].append({"kind": kind, "dims": dims, **kw, "blk": blk, "W": 4,
                           "runs": runs, "vfrac": v})
    # Poiseuille verification (verification.cpp) on the reference, for context
    out["verify"] = []
    for name in ("blk-push-soa", "aa-soa", "list-aa-soa", "list-pull-soa"):
        r = ref.verify(name, 4, 4, 18, g=1e-6, tau=0.9)
        out["verify"].append({"kernel": name, "dims": [4, 4, 18], "steps": r["steps"],
                              "linf_rel": r["linf_rel"], "passed": r["passed"]})
    json.dump(out, open(os.path.join(HERE, "small.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(HERE, "small_snapshots.npz"), **arrays)
    print("wrote small.json", len(out["cases"]), "cases")


CONFIGS = [
    # (id, kernel, kind, dims, extra, steps)
    (1, "blk-push-soa", "channel", (64, 64, 64), {}, 100),
    (2, "list-aa-soa", "channel", (256, 256, 256), {}, 1000),
    (3, "list-pull-soa", "pipe", (512, 256, 256), {"pipe_diameter": 250}, 500),
    (4, "list-aa-soa", "blocks", (400, 400, 400), {"block": 8, "spacing": 8}, 500),
    # cfg 5 needs ~82 GB of host RAM (lattice + snapshot): generated on the
    # GPU box's host (196 GB) with LBMGPU_GOLDEN_OUT=gpurun_out/configs5.json
    (5, "aa-soa", "channel", (1024, 512, 512), {}, 200),
]


def configs(ref: Ref, which):
    path = os.environ.get("LBMGPU_GOLDEN_OUT", os.path.join(HERE, "configs.json"))
    out = json.load(open(path)) if os.path.exists(path) else {}
    for cid, name, kind, dims, extra, steps in CONFIGS:
        if which and cid not in which:
            continue
        t0 = time.time()
        k = ref.kernel(name, kind, *dims, threads=os.cpu_count(), **extra)
        m0 = k.total_mass()
        sec = k.advance(1.0, 3.0 / 16.0, BASE_G, steps)
        snap = k.snapshot()
        n = k.n_fluid
        mid = n // 2
        rec = {"kernel": name, "kind": kind, "dims": list(dims), **extra, "steps": steps,
               "omega_plus": 1.0, "magic_lambda": 3.0 / 16.0, "g": list(BASE_G),
               "n_fluid": n, "fingerprint": f"{ref.fingerprint(snap):016x}",
               "mass0": m0, "mass1": k.total_mass(),
               "sample_node": mid, "sample_pdfs": snap[mid * 19: mid * 19 + 19].tolist(),
               "cpu_seconds": sec, "cpu_threads": os.cpu_count(),
               "cpu_mflups": n * steps / sec / 1e6}
        if name.startswith("list-"):
            for pad in ("auto", "none"):
                for scatter in (False, True):
                    s = ref.structure(kind, *dims, padding=pad, scatter=scatter,
                                      block=extra.get("block", 4), spacing=extra.get("spacing", 4),
                                      pipe_diameter=extra.get("pipe_diameter", 0))
                    rec[f"adj_fnv_{pad}_{'scatter' if scatter else 'gather'}"] = \
                        f"{ref.fingerprint_u32(s['adj']):016x}"
                    rec[f"starts_{pad}"] = [int(v) for v in s["starts"]]
                    rec[f"total_slots_{pad}"] = s["total_slots"]
                    del s
        out[str(cid)] = rec
        del snap, k
        json.dump(out, open(path, "w"), indent=1)
        print(f"cfg {cid}: {rec['fingerprint']} {rec['cpu_mflups']:.2f} MFLUP/s "
              f"({time.time() - t0:.0f} s)", flush=True)


def edge(ref: Ref):
    """Degenerate and ragged shapes (the wrap onto itself of a 1- or 2-cell
    periodic axis, one fluid node, box sizes that are not a multiple of the
    blocks period, a pipe one cell long) for every kernel, and blk tilings
    that do not divide the box: fingerprint + mass after 6 steps."""
    out = {"cases": []}
    cases = [("channel", (1, 3, 3), {}), ("channel", (2, 3, 4), {}), ("slit", (1, 1, 3), {}),
             ("slit", (3, 2, 5), {}), ("pipe", (1, 4, 4), {}), ("pipe", (2, 7, 5), {}),
             ("blocks", (9, 8, 8), dict(block=4, spacing=4)),
             ("blocks", (11, 7, 13), dict(block=3, spacing=2)),
             ("blocks", (5, 5, 5), dict(block=5, spacing=0))]
    for kind, dims, kw in cases:
        for name in ref.kernel_names():
            for blk in ((0, 2, 3) if name.startswith("list-") else (0,)):
                try:
                    k = ref.kernel(name, kind, *dims, threads=2, blk=blk, **kw)
                except Exception as e:  # e.g. no fluid node: ConfigError
                    out["cases"].append({"kernel": name, "kind": kind, "dims": dims, **kw,
                                         "blk": blk, "config_error": str(e)})
                    continue
                init = ref.perturbed(k.n_fluid, 99)
                k.load_state(init)
                k.advance(1.0 / TAU, 3.0 / 16.0, G_TEST, 6)
                out["cases"].append({"kernel": name, "kind": kind, "dims": dims, **kw, "blk": blk,
                                     "seed": 99, "steps": 6, "n_fluid": k.n_fluid,
                                     "fingerprint": f"{k.fingerprint():016x}",
                                     "mass": k.total_mass()})
    json.dump(out, open(os.path.join(HERE, "edge.json"), "w"), indent=1)
    print(len(out["cases"]), "edge cases")


def nodes(ref: Ref):
    """FNV-1a of the reference's node list (order_nodes, list_lattice.cpp:
    123-141; blk = 0) for the list configs, over the int32 little-endian
    (x, y, z) triples -- the bytes lbmgpu_export_structure returns -- added to
    configs.json next to the adjacency FNVs."""
    path = os.path.join(HERE, "configs.json")
    out = json.load(open(path))
    for cid, name, kind, dims, extra, _ in CONFIGS:
        if not name.startswith("list-"):
            continue
        s = ref.structure(kind, *dims, padding="none", scatter=False,
                          block=extra.get("block", 4), spacing=extra.get("spacing", 4),
                          pipe_diameter=extra.get("pipe_diameter", 0))
        nodes = np.ascontiguousarray(s["nodes"], np.int32).view(np.uint32).ravel()
        out[str(cid)]["nodes_fnv"] = f"{ref.fingerprint_u32(nodes):016x}"
        assert f"{ref.fingerprint_u32(s['adj']):016x}" == out[str(cid)]["adj_fnv_none_gather"]
        print(f"cfg {cid}: nodes {out[str(cid)]['nodes_fnv']}", flush=True)
        del s, nodes
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    ref = Ref()
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        small(ref)
    elif what == "edge":
        edge(ref)
    elif what == "nodes":
        nodes(ref)
    else:
        configs(ref, [int(a) for a in sys.argv[2:]])

"""CPU: pin the C restatement oracle (oracle/lbm_oracle.c) to the reference.

The golden fixtures in tests/golden/ were produced by the UNMODIFIED reference
(tests/golden/make_golden.py drives oracle/_ref/liblbm_ref.so, compiled from
/root/reference/proj/src).  The restatement must reproduce them bit for bit;
where the reference library itself is present (this container), it is also
compared directly on extra random cases.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import REF_SO, Q

HERE = os.path.dirname(os.path.abspath(__file__))
TAU = 0.9


def test_restatement_matches_every_golden_case(port, small_golden, small_snapshots):
    """All 17 kernels x 4 geometries (perturbed seed 1234, 8 steps) collapse to
    two families; the port's textbook steppers must equal the reference
    kernels' snapshots bitwise and give the same fingerprints."""
    done = {}
    for case in small_golden["cases"]:
        key = case["snapshot_key"]
        if key not in done:
            fam = key.rsplit("_", 1)[1]
            kw = dict(block=case.get("block", 4), spacing=case.get("spacing", 4))
            _, _, nf = port.geometry(case["kind"], *case["dims"], **kw)
            init = port.perturbed(nf, 1234)
            out, mass = port.run(fam, case["kind"], *case["dims"], case["steps"], 1.0 / TAU,
                                 g=case["g"], init=init, **kw)
            done[key] = (out, mass)
            assert np.array_equal(out, small_snapshots[key]), key
        out, mass = done[key]
        assert f"{port.fingerprint(out):016x}" == case["fingerprint"]
        assert abs(mass - case["mass"]) <= 1e-12 * abs(case["mass"]), case["kernel"]


def test_structures_match_reference(port, small_golden):
    for s in small_golden["structures"]:
        got = port.structure(s["kind"], *s["dims"], block=s.get("block", 4),
                             spacing=s.get("spacing", 4), layout=s["layout"], blk=s["blk"],
                             padding=s["padding"], scatter=s["scatter"])
        assert got["n_fluid"] == s["n_fluid"]
        if s["layout"] == "soa":
            assert [int(v) for v in got["starts"]] == s["starts"]
        assert got["total_slots"] == s["total_slots"]
        assert f"{port.fingerprint(got['adj']):016x}" == s["adj_fnv"], s
        assert f"{port.fingerprint(got['nodes'].reshape(-1).astype(np.uint32)):016x}" == s["nodes_fnv"]


def test_padding_kats(port, small_golden):
    for p in small_golden["padding"]:
        st, tot = port.padding_offsets(p["n_fluid"], p["mode"])
        assert [int(v) for v in st] == p["starts"]
        assert tot == p["total"]


def test_survey_padding_values(port):
    """cfg 2/3/4 starts[1], starts[18], S (pad = auto)."""
    for n, s1, s18, S in [(16516096, 17039568, 306712224, 323228320),
                          (56000000, 56000720, 1014501024, 1070501024)]:
        st, tot = port.padding_offsets(n, "auto")
        assert (int(st[1]), int(st[18]), tot) == (s1, s18, S)


def test_geometry_censuses(port):
    """tests/test_geometry.cpp:10-63 and test_harness.cpp:25-33."""
    assert port.geometry("channel", 500, 100, 100)[2] == 4802000
    assert port.geometry("blocks", 16, 16, 16)[2] == 3584
    assert port.geometry("blocks", 12, 10, 10)[2] == 1136


def test_collide_kats(port):
    """tests/test_d3q19.cpp: equilibrium is a fixed point without force; mass
    and momentum conserved by the collision (force adds g*rho)."""
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    f = port.collide(w, 1.0 / 0.9, port.omega_minus(1.0 / 0.9), (0, 0, 0))
    assert np.max(np.abs(f - w)) <= 1e-16
    rng = np.random.default_rng(7)
    cx = np.array([0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0])
    for _ in range(200):
        f0 = w * (1 + 0.05 * (rng.random(Q) - 0.5))
        f1 = port.collide(f0, 1.3, port.omega_minus(1.3), (1e-5, 0, 0))
        assert abs(f1.sum() - f0.sum()) <= 1e-15
        assert abs((f1 - f0) @ cx - 1e-5 * f0.sum()) <= 1e-15


def test_perturbed_matches_host_mirror(port):
    import paper_1711_11468_b200 as lbm
    for n, seed in [(1, 0), (1136, 1234), (5000, 2**63 + 5)]:
        assert np.array_equal(port.perturbed(n, seed), lbm.perturbed_equilibrium(n, seed))


CONFIGS = os.path.join(HERE, "golden", "configs.json")


def test_config1_fingerprint_from_port(port):
    """The port's full-way textbook stepper reproduces the reference's cfg 1
    fingerprint (channel 64^3, blk-push-soa, 100 steps, omega+=1)."""
    if not os.path.exists(CONFIGS):
        pytest.skip("configs.json missing")
    c = json.load(open(CONFIGS)).get("1")
    if c is None:
        pytest.skip("cfg 1 golden missing")
    out, mass = port.run("full", "channel", 64, 64, 64, 100, 1.0, g=(1e-5, 0, 0))
    assert f"{port.fingerprint(out):016x}" == c["fingerprint"] == "0fc9230302c2fb25"
    assert abs(mass - c["mass1"]) <= 1e-12 * c["mass1"]


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built here")
def test_port_vs_reference_random_cases(port):
    from oracle.oracle import Ref
    ref = Ref()
    rng = np.random.default_rng(11)
    for _ in range(6):
        kind = ["channel", "pipe", "blocks", "slit"][rng.integers(4)]
        dims = tuple(int(v) for v in rng.integers(6, 14, 3))
        kw = dict(block=3, spacing=2) if kind == "blocks" else {}
        seed = int(rng.integers(1 << 30))
        tau = float(rng.uniform(0.55, 1.8))
        g = tuple(float(v) for v in rng.normal(0, 1e-5, 3))
        for name in ("blk-pull-aos", "aa-vec-soa", "list-aa-pv-soa", "list-push-soa"):
            k = ref.kernel(name, kind, *dims, threads=3, **kw)
            init = ref.perturbed(k.n_fluid, seed)
            k.load_state(init)
            k.advance(1.0 / tau, 0.25, g, 6)
            fam = "half" if name.startswith("list-") else "full"
            out, _ = port.run(fam, kind, *dims, 6, 1.0 / tau, 0.25, g=g, init=init, **kw)
            assert np.array_equal(k.snapshot(), out), (name, kind, dims)


def test_restatement_matches_edge_cases(port, edge_golden):
    """Degenerate / ragged shapes (tests/golden/edge.json: 1- and 2-cell
    periodic axes, a single fluid node, blocks boxes that are not a multiple
    of the period, a zero-fluid geometry): the restatement reproduces every
    reference fingerprint and mass, and rejects what the reference rejects."""
    done = {}
    for case in edge_golden["cases"]:
        kw = dict(block=case.get("block", 4), spacing=case.get("spacing", 4))
        if "config_error" in case:
            with pytest.raises(ValueError):
                port.geometry(case["kind"], *case["dims"], **kw)
            continue
        fam = "half" if case["kernel"].startswith("list-") else "full"
        key = (case["kind"], tuple(case["dims"]), kw["block"], kw["spacing"], fam)
        if key not in done:
            _, _, nf = port.geometry(case["kind"], *case["dims"], **kw)
            assert nf == case["n_fluid"]
            init = port.perturbed(nf, case["seed"])
            done[key] = port.run(fam, case["kind"], *case["dims"], case["steps"], 1.0 / TAU,
                                 g=(1e-5, 2e-6, -3e-6), init=init, **kw)
        out, mass = done[key]
        assert f"{port.fingerprint(out):016x}" == case["fingerprint"], case
        assert abs(mass - case["mass"]) <= 1e-12 * abs(case["mass"]), case

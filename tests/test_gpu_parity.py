"""GPU parity tests: the CUDA sweeps (through the C ABI) against the oracle.

Bar: bit-exact PDFs, node lists and adjacency (the reference is built with
-ffp-contract=off and the device collide keeps its expression order with
--fmad=false, so every rounding matches).  Where a check is tolerance based
the tolerance is written in the test: total mass (a compensated device sum
vs a sequential Kahan sum) is compared at 1e-12 relative.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_11468_b200 as lbm  # noqa: E402

TAU = 0.9
G_TEST = (1e-5, 2e-6, -3e-6)  # reference tests/test_kernels.cpp:14-15
PARAMS = lbm.TrtParams.from_tau(TAU)
FORCE = lbm.BodyForce(G_TEST)
NAMES = lbm.kernel_names()


def spec_of(case):
    return lbm.GeometrySpec(case["kind"], *case["dims"], case.get("block", 4), case.get("spacing", 4),
                            case.get("pipe_diameter", 0))


def oracle_state(port, name, kind, dims, steps, seed):
    """The oracle's family stepper (full-way for direct names, half-way for
    list names) from perturbed_equilibrium(seed): the checker the
    decomposition tests compare against directly."""
    _, _, nf = port.geometry(kind, *dims)
    fam = "half" if name.startswith("list-") else "full"
    return port.run(fam, kind, *dims, steps, PARAMS.omega_plus, g=G_TEST,
                    init=port.perturbed(nf, seed))[0]


def test_seventeen_names_and_registry():
    assert len(NAMES) == 17
    with pytest.raises(lbm.ConfigError) as e:
        lbm.make_descriptor("plain-push")
    assert "blk-push-aos" in str(e.value)


@pytest.mark.parametrize("idx", range(68))
def test_kernel_matches_golden_bitwise(idx, small_golden, small_snapshots):
    """Every kernel x {blocks 12x10x10, channel 16x12x10, pipe 9x12x13,
    slit 6x5x9}: perturbed init (seed 1234), 8 steps, tau 0.9,
    g = (1e-5, 2e-6, -3e-6) -- the reference's own recipe
    (tests/test_kernels.cpp:69-94), compared bit for bit."""
    case = small_golden["cases"][idx]
    k = lbm.make_kernel(lbm.make_descriptor(case["kernel"]), spec_of(case))
    assert k.n_fluid() == case["n_fluid"]
    k.load_perturbed(1234)
    host_init = lbm.perturbed_equilibrium(k.n_fluid(), 1234)
    assert np.array_equal(k.snapshot(), host_init)
    k.advance(PARAMS, FORCE, case["steps"])
    snap = k.snapshot()
    expect = small_snapshots[case["snapshot_key"]]
    assert np.array_equal(snap, expect), case["kernel"]
    assert f"{lbm.state_fingerprint(snap):016x}" == case["fingerprint"]
    assert f"{k.fingerprint():016x}" == case["fingerprint"]
    assert abs(k.total_mass() - case["mass"]) <= 1e-12 * abs(case["mass"])


@pytest.mark.parametrize("fused", ["default", "per-sweep"])
@pytest.mark.parametrize("name", NAMES)
def test_against_port_oracle_steppers(name, fused, port, monkeypatch):
    """Host load_state path + several geometries, against our C restatement
    of the reference steppers (tests/support/reference.hpp:33-105).  Small
    direct lattices normally run as one fused grid-barrier launch; the
    per-sweep kernels (used for large lattices) are forced with
    LBMGPU_FUSED_MB=0, so every path is checked bit for bit.  channel
    32x12x8 takes the AoS 3-D halo-tile sweeps (nx % 16, ny and nz % 4),
    the other two boxes the per-node AoS kernels."""
    if fused == "per-sweep":
        monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    for kind, dims in [("blocks", (12, 12, 12)), ("channel", (33, 7, 9)),
                       ("channel", (32, 12, 8))]:
        _, _, nf = port.geometry(kind, *dims)
        init = port.perturbed(nf, 99)
        fam = "half" if name.startswith("list-") else "full"
        for steps in (6, 7) if not name.startswith(("aa", "list-aa")) else (6,):
            expect, _ = port.run(fam, kind, *dims, steps, PARAMS.omega_plus, g=G_TEST, init=init)
            k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims))
            k.load_state(init)
            k.advance(PARAMS, FORCE, steps)
            got = k.snapshot()
            assert port.max_rel_diff(got, expect) <= 1e-12, (name, kind)
            assert np.array_equal(got, expect), (name, kind, steps)
            # a second advance continues from the swapped buffers correctly
            k.advance(PARAMS, FORCE, 2)
            expect2, _ = port.run(fam, kind, *dims, steps + 2, PARAMS.omega_plus, g=G_TEST,
                                  init=init)
            assert np.array_equal(k.snapshot(), expect2), (name, kind, steps + 2)


@pytest.mark.parametrize("kind,dims", [("channel", (16, 12, 10)), ("blocks", (24, 20, 20)),
                                       ("pipe", (9, 12, 13))])
def test_ria_codings_bitwise_equal(kind, dims, monkeypatch):
    """Every coding of the run-coded odd step -- run table (0), group
    patterns (1), per-node pattern ids (2: 8/16/32-bit ids for <= 256 /
    65,536 / 2^20 distinct run patterns), auto (-1) -- is bitwise
    list-aa-soa."""
    spec = lbm.GeometrySpec(kind, *dims)
    ref = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec)
    ref.load_perturbed(21)
    ref.advance(PARAMS, FORCE, 10)
    for mode in ("0", "1", "2", "-1"):
        monkeypatch.setenv("LBMGPU_RIA_MODE", mode)
        for name in ("list-aa-ria-soa", "list-aa-pv-soa"):
            k = lbm.make_kernel(lbm.make_descriptor(name), spec)
            k.load_perturbed(21)
            k.advance(PARAMS, FORCE, 10)
            assert k.fingerprint() == ref.fingerprint(), (mode, name)
            del k


@pytest.mark.parametrize("name", ["list-pull-soa", "list-pull-split-nt-1s-soa"])
@pytest.mark.parametrize("kind,dims", [("channel", (16, 12, 10)), ("pipe", (16, 14, 13)),
                                       ("blocks", (24, 24, 24)), ("slit", (6, 5, 9))])
def test_list_pull_pattern_ids_bitwise(name, kind, dims, monkeypatch):
    """LBMGPU_PULL_PID=1: the one-step pull gathers through pattern ids of
    its Gather table (the RIA coding applied to the pull); bitwise equal to
    the indexed pull, odd and even step counts."""
    spec = lbm.GeometrySpec(kind, *dims)
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    for steps in (5, 4):
        ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
        ref.load_perturbed(31)
        ref.advance(PARAMS, FORCE, steps)
        monkeypatch.setenv("LBMGPU_PULL_PID", "1")
        k = lbm.make_kernel(lbm.make_descriptor(name), spec)
        monkeypatch.delenv("LBMGPU_PULL_PID")
        k.load_perturbed(31)
        k.kernel_stats_enable(True)
        k.advance(PARAMS, FORCE, steps)
        assert any(n.startswith("list_pull_pid") for n in k.kernel_stats())
        assert k.fingerprint() == ref.fingerprint(), (name, steps)


@pytest.mark.parametrize("dims,expect", [((16, 12, 10, 4, 4), "list_aa_odd_ria_pid_soa"),
                                         ((24, 24, 24, 4, 4), "list_aa_odd_ria_pid16_soa"),
                                         ((192, 192, 192, 4, 4), "list_aa_odd_ria_pid32_soa")])
def test_ria_pattern_id_widths(dims, expect):
    """Pattern ids of every width: blocks 24^3 has 1,386 distinct run
    patterns (16-bit ids), blocks 192^3 has 77,553 (32-bit ids; cfg 4 has
    144,084 -- counts from tools/ria_patterns.py).  Auto mode picks the
    width; bitwise list-aa-soa."""
    kind = "channel" if dims[0] == 16 else "blocks"
    spec = lbm.GeometrySpec(kind, *dims)
    ref = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec)
    ref.load_perturbed(23)
    ref.advance(PARAMS, FORCE, 6)
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-ria-soa"), spec)
    k.load_perturbed(23)
    k.kernel_stats_enable(True)
    k.advance(PARAMS, FORCE, 6)
    assert expect in k.kernel_stats()
    assert k.fingerprint() == ref.fingerprint()


@pytest.mark.parametrize("name", ["blk-pull-aos", "blk-push-aos", "aa-aos"])
@pytest.mark.parametrize("kind,dims", [("channel", (16, 8, 8)), ("channel", (32, 12, 8)),
                                       ("blocks", (32, 16, 16)), ("slit", (48, 4, 12)),
                                       ("pipe", (16, 12, 12)),
                                       # boxes with interior tiles (no wrapped neighbour:
                                       # the fixed-offset fast path) beside surface tiles
                                       ("channel", (64, 16, 16)), ("blocks", (48, 12, 20)),
                                       ("pipe", (80, 20, 12))])
def test_aos_halo_tiles_against_oracle(name, kind, dims, port, monkeypatch):
    """The AoS 3-D halo-tile sweeps (TMA row copies split at the x wrap,
    y / z wrap of the halo rows, bulk stores of whole destination records)
    against the oracle's family stepper, bit for bit: blk-pull-aos and
    blk-push-aos (which runs the push mapping in pull order: collide pass,
    gather sweeps, stream-only pass -- reference tests/test_kernels.cpp:
    96-126) over odd and even step counts and repeated advance(1) calls, and
    aa-aos (odd step gathers through the tiles)."""
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    _, _, nf = port.geometry(kind, *dims)
    init = port.perturbed(nf, 17)
    k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims))
    k.load_state(init)
    k.kernel_stats_enable(True)
    runs = [6, 2] if name.startswith("aa") else [5, 2, 1, 1]
    done = 0
    for st in runs:
        k.advance(PARAMS, FORCE, st)
        done += st
        expect, _ = port.run("full", kind, *dims, done, PARAMS.omega_plus, g=G_TEST, init=init)
        assert np.array_equal(k.snapshot(), expect), (name, kind, dims, done)
    rows = set(k.kernel_stats())
    tile = {"blk-pull-aos": "full_pull_aos", "blk-push-aos": "full_push_aos",
            "aa-aos": "full_aa_odd_aos"}[name]
    assert tile in rows, rows


@pytest.mark.parametrize("by", ["0", "1", "2", "3", "4", "16"])
def test_aos_tile_traversal_orders_against_oracle(by, port, monkeypatch):
    """The 3-D grid of the AoS tile kernels in every traversal order
    (LBMGPU_TILE_BY: plain, blocks of 2 / 4 y tiles, and the values that fall
    back to plain -- not a power of two, not dividing the y tile count) on a
    box with interior and surface tiles, bit for bit against the oracle."""
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    monkeypatch.setenv("LBMGPU_TILE_BY", by)
    kind, dims = "blocks", (64, 16, 12)
    _, _, nf = port.geometry(kind, *dims)
    init = port.perturbed(nf, 29)
    expect, _ = port.run("full", kind, *dims, 4, PARAMS.omega_plus, g=G_TEST, init=init)
    for name in ("aa-aos", "blk-pull-aos", "blk-push-aos"):
        k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims))
        k.load_state(init)
        k.advance(PARAMS, FORCE, 4)
        assert np.array_equal(k.snapshot(), expect), (name, by)


LIST_AOS_TILE_CASES = [
    ("channel", (16, 12, 10)), ("channel", (9, 7, 13)), ("blocks", (12, 10, 10)),
    ("blocks", (20, 18, 22)), ("pipe", (9, 12, 13)), ("slit", (6, 5, 9)),
    ("channel", (5, 6, 34)), ("channel", (3, 4, 6)), ("blocks", (8, 9, 11)), ("slit", (4, 3, 40)),
    ("channel", (64, 64, 64)), ("blocks", (40, 36, 44)),  # persistent CTAs: several tiles each
]


@pytest.mark.parametrize("shape", ["0", "1", "5", "12"])
@pytest.mark.parametrize("kind,dims", LIST_AOS_TILE_CASES)
def test_list_aa_aos_staging_tiles_against_oracle(shape, kind, dims, port, monkeypatch):
    """list-aa-aos odd step through the 3-D staging tiles
    (list_aos_tile.cuh) for every instantiated tile shape (LBMGPU_LTILE):
    ragged boxes that no tile divides, rows shorter than the staged z range,
    z ranges wrapping periodically onto one and two list ranges, tiles wider
    than the box (halo rows wrapping onto own rows), solid obstacles inside
    the staged rows -- bit for bit against the oracle's half-way stepper
    (kernels_list_aa.cpp:22-31) over repeated advance calls."""
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    monkeypatch.setenv("LBMGPU_LTILE", shape)
    _, _, nf = port.geometry(kind, *dims)
    init = port.perturbed(nf, 23)
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-aos"), lbm.GeometrySpec(kind, *dims))
    k.load_state(init)
    k.kernel_stats_enable(True)
    done = 0
    for st in (4, 2):
        k.advance(PARAMS, FORCE, st)
        done += st
        expect, _ = port.run("half", kind, *dims, done, PARAMS.omega_plus, g=G_TEST, init=init)
        assert np.array_equal(k.snapshot(), expect), (shape, kind, dims, done)
    assert "list_aa_odd_aos" in k.kernel_stats()


RUN_JOB_CASES = [
    # (kind, dims, steps, JOB_SLABS, JOB_CHUNK, JOB_CHUNK_OUT, pipelined for aa-soa)
    ("channel", (16, 12, 10), 6, "512", "16", "32", True),   # the defaults
    ("channel", (32, 12, 40), 10, "7", "2", "3", True),      # ragged slabs and chunks
    ("channel", (24, 16, 67), 12, "3", "1", "1", True),      # fewer slabs than steps
    ("channel", (16, 8, 130), 4, "128", "4", "9", True),     # more slabs than steps
    ("slit", (6, 5, 37), 8, "5", "3", "2", True),
    ("channel", (32, 16, 33), 2, "1", "1", "1", True),       # one slab, one chunk
    ("channel", (40, 8, 24), 6, "512", "1", "64", True),     # chunk wider than the box
    ("pipe", (9, 12, 13), 4, "512", "16", "32", False),      # columns differ: plain sequence
    ("blocks", (12, 10, 10), 4, "512", "16", "32", False),   # periodic z, obstacles: plain
]


@pytest.mark.parametrize("name", ["aa-soa", "aa-vec-soa", "aa-aos", "blk-push-soa", "list-aa-soa"])
@pytest.mark.parametrize("kind,dims,steps,slabs,chunk,chunk_out,piped", RUN_JOB_CASES)
def test_run_job_equals_load_advance_snapshot(name, kind, dims, steps, slabs, chunk, chunk_out,
                                              piped, port, monkeypatch):
    """lbmgpu_run (load_state + advance + snapshot in one call, host
    transfers pipelined with diagonal-round sweeps over z slabs where the
    lattice allows) is bitwise the three separate calls and the oracle, for
    page-locked and for pageable buffers, in place (out aliases in) or not;
    the pipelined schedule runs exactly where documented."""
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")  # small boxes: per-sweep launches
    monkeypatch.setenv("LBMGPU_JOB_SLABS", slabs)
    monkeypatch.setenv("LBMGPU_JOB_CHUNK", chunk)
    monkeypatch.setenv("LBMGPU_JOB_CHUNK_OUT", chunk_out)
    spec = lbm.GeometrySpec(kind, *dims)
    _, _, nf = port.geometry(kind, *dims)
    init = port.perturbed(nf, 41)
    fam = "half" if name.startswith("list-") else "full"
    expect, _ = port.run(fam, kind, *dims, steps, PARAMS.omega_plus, g=G_TEST, init=init)
    ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
    ref.load_state(init)
    ref.advance(PARAMS, FORCE, steps)
    plain = ref.snapshot()
    assert np.array_equal(plain, expect)
    k = lbm.make_kernel(lbm.make_descriptor(name), spec)
    bin_, bout = lbm.PinnedBuffer(nf * 19), lbm.PinnedBuffer(nf * 19)
    bin_.array[:] = init
    out, pipelined = k.run(bin_.array, PARAMS, FORCE, steps, out=bout.array)
    assert pipelined == (piped and name in ("aa-soa", "aa-vec-soa"))
    assert np.array_equal(out, expect), (name, kind, dims)
    # again from the result, in place (out aliases in): 2 * steps in all
    out2, _ = k.run(bout.array, PARAMS, FORCE, steps, out=bout.array)
    ref.advance(PARAMS, FORCE, steps)
    assert np.array_equal(out2, ref.snapshot())
    # pageable buffers: always the plain sequence, same result (a fresh
    # lattice: load_state writes fluid nodes only, and the solid records of
    # a full lattice carry the populations in flight -- as in the reference,
    # full_lattice.cpp:88-100)
    k3 = lbm.make_kernel(lbm.make_descriptor(name), spec)
    out3, p3 = k3.run(init, PARAMS, FORCE, steps)
    assert not p3 and np.array_equal(out3, expect)
    bin_.free()
    bout.free()


def test_run_job_validation():
    """lbmgpu_run validates like load_state / advance / snapshot."""
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 16, 12, 10))
    n = k.n_fluid() * 19
    with pytest.raises(lbm.ConfigError) as e:
        k.run(np.zeros(n - 1), PARAMS, FORCE, 2)
    assert "state size" in str(e.value)
    with pytest.raises(lbm.ConfigError) as e:
        k.run(np.zeros(n), PARAMS, FORCE, 3)
    assert "even step count" in str(e.value)
    with pytest.raises(lbm.ConfigError):
        k.run(np.zeros(n), lbm.TrtParams(2.5), FORCE, 2)


def test_no_out_of_bounds_writes_guard_zones(monkeypatch):
    """Memory-safety check in place of compute-sanitizer (closed on this
    pool): with LBMGPU_GUARD=1 every device buffer carries 4 KiB guard zones
    of a fixed byte pattern; after every kernel family has run -- each name
    per-sweep and fused, the TMA tiles and 3-D halo tiles, RIA codings,
    z-slab and node-range decompositions with every transport (device
    copies, NCCL, peer memory), the pipelined job,
    snapshot / load / verify -- no guard byte may have changed."""
    monkeypatch.setenv("LBMGPU_GUARD", "1")
    assert lbm.lbmgpu.guard_selftest() == 1  # a planted 8-byte overrun is seen
    small = lbm.GeometrySpec("blocks", 12, 10, 10)
    tiled = lbm.GeometrySpec("channel", 32, 12, 8)  # nx % 16, ny/nz % 4: halo tiles
    keep = []
    for fused in ("96", "0"):
        monkeypatch.setenv("LBMGPU_FUSED_MB", fused)
        for name in lbm.kernel_names():
            for spec in (small, tiled):
                k = lbm.make_kernel(lbm.make_descriptor(name, blk=2 if "list" in name else 0), spec)
                k.load_perturbed(3)
                k.advance(PARAMS, FORCE, 6)
                k.load_state(k.snapshot())
                k.total_mass()
                keep.append(k)
    monkeypatch.setenv("LBMGPU_FUSED_MB", "0")
    # direct AoS tiles with interior tiles (fixed-offset fast path) in every
    # traversal order, beside the surface tiles
    for by in ("8", "0", "2"):
        monkeypatch.setenv("LBMGPU_TILE_BY", by)
        for name in ("aa-aos", "blk-pull-aos", "blk-push-aos"):
            k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec("blocks", 64, 16, 12))
            k.load_perturbed(3)
            k.advance(PARAMS, FORCE, 4)
            keep.append(k)
    monkeypatch.delenv("LBMGPU_TILE_BY")
    # the pipelined job (staging buffers, layout kernels, slab launches)
    for slabs, chunk, chunk_out in (("512", "16", "32"), ("7", "2", "3")):
        monkeypatch.setenv("LBMGPU_JOB_SLABS", slabs)
        monkeypatch.setenv("LBMGPU_JOB_CHUNK", chunk)
        monkeypatch.setenv("LBMGPU_JOB_CHUNK_OUT", chunk_out)
        k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 32, 12, 40))
        buf = lbm.PinnedBuffer(k.n_fluid() * 19)
        buf.array[:] = lbm.perturbed_equilibrium(k.n_fluid(), 3)
        _, piped = k.run(buf.array, PARAMS, FORCE, 6, out=buf.array)
        assert piped
        buf.free()
        keep.append(k)
    for shape in ("0", "1", "5", "12"):  # list-aa-aos staging tiles (blk = 0)
        monkeypatch.setenv("LBMGPU_LTILE", shape)
        for spec in (small, tiled, lbm.GeometrySpec("pipe", 9, 12, 13)):
            k = lbm.make_kernel(lbm.make_descriptor("list-aa-aos"), spec)
            k.load_perturbed(3)
            k.advance(PARAMS, FORCE, 4)
            keep.append(k)
    monkeypatch.delenv("LBMGPU_LTILE")
    for mode in ("0", "1", "2"):
        monkeypatch.setenv("LBMGPU_RIA_MODE", mode)
        k = lbm.make_kernel(lbm.make_descriptor("list-aa-ria-soa"), small)
        k.advance(PARAMS, FORCE, 4)
        keep.append(k)
    for name in ("aa-soa", "blk-push-soa", "blk-pull-soa"):
        for extra in ({}, {"nccl_id": lbm.lbmgpu.nccl_unique_id()}, {"transport": "peer"}):
            k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec("channel", 16, 12, 24),
                                dist={"virtual_parts": 3, **extra})
            k.advance(PARAMS, FORCE, 4)
            k.snapshot_local()
            keep.append(k)
    for extra in ({}, {"nccl_id": lbm.lbmgpu.nccl_unique_id()}):
        k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("blocks", 16, 16, 16),
                            dist={"virtual_parts": 3, **extra})
        k.advance(PARAMS, FORCE, 4)
        k.snapshot()
        keep.append(k)
    # peer transport over the z ring (blocks)
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("blocks", 16, 16, 16),
                        dist={"virtual_parts": 4, "transport": "peer"})
    k.advance(PARAMS, FORCE, 4)
    keep.append(k)
    rep = lbm.verify_kernel(lbm.make_descriptor("aa-soa"))
    assert rep["passed"]
    bad, msg = lbm.lbmgpu.guard_check()
    assert bad == 0, msg
    del keep


def test_edge_shapes_match_reference(edge_golden):
    """Degenerate and ragged shapes for every kernel (tests/golden/edge.json,
    generated by the reference): 1- and 2-cell periodic axes that wrap onto
    themselves, a single fluid node, blocks boxes that are not a multiple of
    the period, blk tilings that do not divide the box; fingerprint and mass
    equal, and a zero-fluid geometry rejected with the reference's error."""
    for case in edge_golden["cases"]:
        spec = lbm.GeometrySpec(case["kind"], *case["dims"], case.get("block", 4),
                                case.get("spacing", 4))
        desc = lbm.make_descriptor(case["kernel"], blk=case["blk"])
        if "config_error" in case:
            with pytest.raises(lbm.ConfigError) as e:
                lbm.make_kernel(desc, spec)
            assert "produced no fluid nodes" in str(e.value)
            continue
        k = lbm.make_kernel(desc, spec)
        assert k.n_fluid() == case["n_fluid"]
        k.load_perturbed(case["seed"])
        k.advance(PARAMS, FORCE, case["steps"])
        assert f"{k.fingerprint():016x}" == case["fingerprint"], case
        assert abs(k.total_mass() - case["mass"]) <= 1e-12 * abs(case["mass"]), case
        del k


@pytest.mark.parametrize("name", ["blk-push-soa", "blk-pull-soa", "aa-soa", "blk-push-aos",
                                  "aa-aos"])
@pytest.mark.parametrize("kind,dims", [("channel", (64, 64, 64)), ("blocks", (48, 40, 36))])
def test_fused_launch_equals_per_sweep_at_scale(name, kind, dims, monkeypatch):
    """The multi-sweep grid-barrier launch at a cfg-1-sized lattice, where
    hundreds of blocks race through 21 sweeps (odd count for push/pull), is
    bitwise the per-sweep kernels' result."""
    steps = 20 if name.startswith("aa") else 21
    res = []
    for mb in (None, "0"):
        if mb is not None:
            monkeypatch.setenv("LBMGPU_FUSED_MB", mb)
        k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims))
        k.load_perturbed(7)
        k.advance(PARAMS, FORCE, steps)
        k.advance(PARAMS, FORCE, 4)
        res.append(k.fingerprint())
        del k
    assert len(set(res)) == 1, (name, kind, [f"{r:016x}" for r in res])


@pytest.mark.parametrize("name", ["list-aa-soa", "list-pull-soa", "list-push-soa", "list-aa-aos",
                                  "list-pull-aos"])
@pytest.mark.parametrize("kind,dims", [("channel", (64, 64, 64)), ("blocks", (48, 40, 36))])
def test_list_fused_launch_equals_per_sweep_at_scale(name, kind, dims, monkeypatch):
    """The fused multi-sweep list launch on a cfg-1-sized lattice (hundreds
    of blocks racing through 21 sweeps, grid sync between them) is bitwise
    the per-sweep kernels' result."""
    steps = 20 if "-aa-" in name else 21
    res = []
    for mb in (None, "0"):
        if mb is not None:
            monkeypatch.setenv("LBMGPU_FUSED_MB", mb)
        k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims))
        k.load_perturbed(8)
        k.advance(PARAMS, FORCE, steps)
        k.advance(PARAMS, FORCE, 4)
        res.append(k.fingerprint())
        del k
    assert res[0] == res[1], (name, kind, [f"{r:016x}" for r in res])


def _list_kernel_for(layout, scatter):
    if scatter:
        return "list-aa-soa" if layout == "soa" else "list-aa-aos"
    return "list-pull-soa" if layout == "soa" else "list-pull-aos"


@pytest.mark.parametrize("idx", range(84))
def test_list_structure_bit_exact(idx, small_golden, port):
    """Node order, slot starts and adjacency exported from the device builder
    == the reference build_structure (list_lattice.cpp:149-204), for
    blk 0/2/3, padding none/auto/thrash, gather/scatter, SoA/AoS."""
    if idx >= len(small_golden["structures"]):
        pytest.skip("fewer structure cases")
    s = small_golden["structures"][idx]
    name = _list_kernel_for(s["layout"], s["scatter"])
    k = lbm.make_kernel(lbm.make_descriptor(name, blk=s["blk"]), spec_of(s),
                        lbm.PaddingPolicy(s["padding"]))
    nodes, adj, starts, total = k.export_structure()
    assert [int(v) for v in starts] == (s["starts"] if s["layout"] == "soa" else [0] * 19)
    assert total == s["total_slots"]
    assert f"{port.fingerprint(adj):016x}" == s["adj_fnv"]
    assert f"{port.fingerprint(nodes.reshape(-1).astype(np.uint32)):016x}" == s["nodes_fnv"]


def test_structure_against_port_builder(port):
    for kind, dims, kw in [("pipe", (5, 14, 11), {}), ("blocks", (10, 9, 11), dict(block=3, spacing=2))]:
        for blk in (0, 4):
            for scatter in (False, True):
                ref = port.structure(kind, *dims, blk=blk, scatter=scatter, **kw)
                name = _list_kernel_for("soa", scatter)
                k = lbm.make_kernel(lbm.make_descriptor(name, blk=blk),
                                    lbm.GeometrySpec(kind, *dims, kw.get("block", 4), kw.get("spacing", 4)))
                nodes, adj, starts, total = k.export_structure()
                assert np.array_equal(nodes, ref["nodes"])
                assert np.array_equal(adj, ref["adj"])
                assert np.array_equal(starts, ref["starts"])


def test_blocking_and_padding_never_change_results():
    """tests/test_kernels.cpp:197-241 on the GPU."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    base = {}
    for name in ("blk-push-aos", "aa-vec-soa", "list-aa-pv-soa", "list-pull-soa", "list-aa-soa",
                 "list-pull-split-nt-1s-soa"):
        for blk in (0, 2, 8, 50):
            for pad in ("none", "auto", "thrash"):
                k = lbm.make_kernel(lbm.make_descriptor(name, blk=blk), spec, lbm.PaddingPolicy(pad))
                k.load_perturbed(8)
                k.advance(PARAMS, FORCE, 8)
                s = k.snapshot()
                if name not in base:
                    base[name] = s
                else:
                    assert np.array_equal(s, base[name]), (name, blk, pad)


def test_equilibrium_fixed_point_every_kernel():
    """tests/test_kernels.cpp:56-67."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    for name in NAMES:
        k = lbm.make_kernel(lbm.make_descriptor(name), spec)
        k.advance(PARAMS, lbm.BodyForce(), 4)
        s = k.snapshot().reshape(-1, 19)
        assert np.max(np.abs(s - w)) <= 1e-15, name


def test_push_equals_pull_and_aa_pair_equals_two_steps():
    """tests/test_kernels.cpp:96-126."""
    spec = lbm.GeometrySpec("blocks", 12, 12, 12)
    for a, b in (("blk-push-soa", "blk-pull-soa"), ("list-push-aos", "list-pull-aos")):
        ka = lbm.make_kernel(lbm.make_descriptor(a), spec)
        kb = lbm.make_kernel(lbm.make_descriptor(b), spec)
        for k in (ka, kb):
            k.load_perturbed(99)
            k.advance(PARAMS, FORCE, 1)
        assert np.array_equal(ka.snapshot(), kb.snapshot())
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    os_k = lbm.make_kernel(lbm.make_descriptor("blk-push-soa"), spec)
    aa_k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), spec)
    for k in (os_k, aa_k):
        k.load_perturbed(5)
        k.advance(PARAMS, FORCE, 2)
    assert np.array_equal(os_k.snapshot(), aa_k.snapshot())


def test_advance_zero_composition_and_rejections():
    """tests/test_kernels.cpp:146-175."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    for name in ("blk-pull-aos", "list-aa-soa", "aa-soa", "list-pull-soa"):
        a = lbm.make_kernel(lbm.make_descriptor(name), spec)
        a.load_perturbed(3)
        init = a.snapshot()
        a.advance(PARAMS, FORCE, 0)
        assert np.array_equal(a.snapshot(), init)
        a.advance(PARAMS, FORCE, 4)
        b = lbm.make_kernel(lbm.make_descriptor(name), spec)
        b.load_state(init)
        b.advance(PARAMS, FORCE, 2)
        b.advance(PARAMS, FORCE, 2)
        assert np.array_equal(a.snapshot(), b.snapshot())
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec)
    before = k.snapshot()
    with pytest.raises(lbm.ConfigError):
        k.advance(PARAMS, FORCE, 3)
    assert np.array_equal(k.snapshot(), before)
    with pytest.raises(lbm.ConfigError):
        k.advance(PARAMS, FORCE, -2)
    with pytest.raises(lbm.ConfigError):
        k.advance(lbm.TrtParams(2.5), FORCE, 2)
    with pytest.raises(lbm.ConfigError):
        k.load_state(np.zeros(5))


def test_mass_conserved_without_forcing():
    """tests/test_kernels.cpp:243-256: |dm| <= 1e-11 m over 100 steps."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    for name in NAMES:
        k = lbm.make_kernel(lbm.make_descriptor(name), spec)
        k.load_perturbed(21)
        m0 = k.total_mass()
        k.advance(PARAMS, lbm.BodyForce(), 100)
        assert abs(k.total_mass() - m0) <= 1e-11 * m0, name


def test_ria_stats_match_reference(small_golden):
    for r in small_golden["ria"]:
        k = lbm.make_kernel(lbm.make_descriptor("list-aa-pv-soa", blk=r["blk"], vector_width=r["W"]),
                            spec_of(r), lbm.PaddingPolicy.none())
        st = k.ria_stats()
        assert st["total_runs"] == r["runs"]
        assert k.vector_fraction() == r["vfrac"]
        assert k.pv_chunk_fraction() == r["vfrac"]
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("channel", 20, 10, 10))
    assert k.ria_stats() is None and k.vector_fraction() is None


def test_capabilities():
    spec = lbm.GeometrySpec("blocks", 12, 10, 10)
    assert lbm.make_kernel(lbm.make_descriptor("list-pull-split-nt-1s-soa"), spec).capabilities().nt_streams_effective == 1
    assert lbm.make_kernel(lbm.make_descriptor("list-pull-split-nt-2s-soa"), spec).capabilities().nt_streams_effective == 2
    assert lbm.make_kernel(lbm.make_descriptor("blk-push-soa"), spec).capabilities().nt_streams_effective == 0


@pytest.mark.parametrize("name", ["aa-soa", "blk-push-soa", "blk-pull-soa"])
@pytest.mark.parametrize("kind,dims,parts", [
    ("channel", (16, 12, 24), 2), ("channel", (16, 12, 24), 3), ("channel", (16, 12, 24), 4),
    ("channel", (33, 10, 17), 5), ("blocks", (12, 10, 16), 2), ("blocks", (12, 10, 16), 4),
    ("slit", (6, 5, 9), 3), ("pipe", (9, 12, 13), 13)])
def test_zslab_parts_bitwise_equal_single(name, kind, dims, parts, port):
    """z-slab decomposition (the multi-GPU plan, emulated on one device):
    state bitwise the oracle's and the single-part run's for 1..N parts --
    the worker-count invariance of tests/test_kernels.cpp:177-195 carried to
    the slab split.  AA: halo phases 0/1; one-step push / pull: phases 2/3
    with the z ring (solid nodes stream too), down to one plane per slab;
    odd step counts leave push/pull on the second grid."""
    spec = lbm.GeometrySpec(kind, *dims)
    steps = (4, 6) if name.startswith("aa") else (3, 6)
    ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
    ref.load_perturbed(4242)
    ref.advance(PARAMS, FORCE, sum(steps))
    k = lbm.make_kernel(lbm.make_descriptor(name), spec, dist={"virtual_parts": parts})
    k.load_perturbed(4242)
    init = k.snapshot()
    assert np.array_equal(init, lbm.perturbed_equilibrium(k.n_fluid(), 4242))
    for st in steps:
        k.advance(PARAMS, FORCE, st)
    assert np.array_equal(k.snapshot(), oracle_state(port, name, kind, dims, sum(steps), 4242))
    assert np.array_equal(k.snapshot(), ref.snapshot()), name
    assert abs(k.total_mass() - ref.total_mass()) <= 1e-12 * ref.total_mass()


@pytest.mark.parametrize("name", ["aa-soa", "blk-push-soa", "blk-pull-soa"])
@pytest.mark.parametrize("kind,dims,parts", [("channel", (32, 12, 24), 3), ("blocks", (16, 16, 16), 2)])
def test_zslab_nccl_transport_single_gpu(name, kind, dims, parts, port):
    """The NCCL halo transport (grouped ncclSend/ncclRecv on a comm stream,
    event-ordered against the compute stream) exercised on one GPU: one NCCL
    rank owning all slabs, self send/recv per plan row.  Bitwise equal to the
    single-slab run."""
    spec = lbm.GeometrySpec(kind, *dims)
    ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
    ref.load_perturbed(31)
    ref.advance(PARAMS, FORCE, 8)
    k = lbm.make_kernel(lbm.make_descriptor(name), spec,
                        dist={"virtual_parts": parts, "nccl_id": lbm.lbmgpu.nccl_unique_id()})
    k.load_perturbed(31)
    k.advance(PARAMS, FORCE, 8)
    assert np.array_equal(k.snapshot(), oracle_state(port, name, kind, dims, 8, 31))
    assert np.array_equal(k.snapshot(), ref.snapshot())
    assert abs(k.total_mass() - ref.total_mass()) <= 1e-12 * ref.total_mass()


@pytest.mark.parametrize("name", ["aa-soa", "aa-vec-soa", "blk-push-soa", "blk-pull-soa"])
@pytest.mark.parametrize("kind,dims,parts", [
    ("channel", (16, 12, 24), 2), ("channel", (33, 10, 17), 5), ("blocks", (12, 10, 16), 2),
    ("blocks", (12, 10, 16), 4), ("slit", (6, 5, 9), 3), ("pipe", (9, 12, 13), 13),
    ("blocks", (16, 16, 16), 16)])
def test_zslab_peer_transport_bitwise_equal_single(name, kind, dims, parts, port):
    """Peer-memory transport (direct_peer.cuh): no halo copy at all -- the
    AA boundary planes' odd sub-step loads and stores the neighbour slab's
    slots, the pull's boundary gathers read the neighbour's source grid,
    the push's boundary stores land in the neighbour's destination grid
    (slot chosen by the solid-target mask, no staging / merge); epoch flags
    in the neighbour's memory order the sub-steps.  Emulated with all slabs
    on one device (device pointers instead of CUDA IPC mappings; the flag
    protocol runs unchanged).  Covers the z ring (blocks: fluid on z = 0;
    one-step kernels always), two slabs with the ring (lower == upper
    neighbour), one plane per slab (pipe 13, blocks 16) and odd step counts
    (push / pull end on the second grid).  Bitwise equal to the single-slab
    run, over several advance() calls, total mass included."""
    spec = lbm.GeometrySpec(kind, *dims)
    aa = name.startswith("aa")
    steps = (4, 2, 4) if aa else (3, 2, 4)
    ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
    ref.load_perturbed(777)
    ref.advance(PARAMS, FORCE, sum(steps))
    k = lbm.make_kernel(lbm.make_descriptor(name), spec,
                        dist={"virtual_parts": parts, "transport": "peer"})
    k.load_perturbed(777)
    k.kernel_stats_enable(True)
    for st in steps:
        k.advance(PARAMS, FORCE, st)
    assert np.array_equal(k.snapshot(), oracle_state(port, name, kind, dims, sum(steps), 777))
    assert np.array_equal(k.snapshot(), ref.snapshot()), name
    assert abs(k.total_mass() - ref.total_mass()) <= 1e-12 * ref.total_mass()
    names = set(k.kernel_stats())
    peer_kernel = {"aa-soa": "full_aa_odd_soa_peer", "aa-vec-soa": "full_aa_odd_soa_peer",
                   "blk-push-soa": "full_push_soa_peer", "blk-pull-soa": "full_pull_soa_peer"}
    assert peer_kernel[name] in names and "peer_wait" in names
    assert "push_halo_merge" not in names


def test_zslab_peer_transport_errors():
    spec = lbm.GeometrySpec("channel", 16, 12, 24)
    with pytest.raises(lbm.ConfigError, match="peer transport"):
        lbm.make_kernel(lbm.make_descriptor("aa-soa"), spec, dist={"transport": "peer"})
    with pytest.raises(lbm.ConfigError, match="peer transport"):
        lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec,
                        dist={"virtual_parts": 2, "transport": "peer"})
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), spec,
                        dist={"virtual_parts": 3, "transport": "peer"})
    with pytest.raises(lbm.ConfigError, match="nranks > 1"):
        k.peer_export()


@pytest.mark.parametrize("name", ["list-aa-soa", "list-aa-aos"])
@pytest.mark.parametrize("kind,dims,parts", [
    ("channel", (20, 12, 10), 2), ("channel", (20, 12, 10), 3), ("channel", (20, 12, 10), 4),
    ("blocks", (16, 16, 16), 2), ("blocks", (16, 16, 16), 5), ("pipe", (12, 14, 13), 4),
    ("blocks", (12, 10, 10), 3)])
def test_list_node_range_parts_bitwise(name, kind, dims, parts, port):
    """List AA decomposed into contiguous node ranges (x-slabs for blk = 0,
    the split of reference kernels_list_aa.cpp:63-74) with index-list halos
    (SURVEY 8(f) row 2), emulated on one GPU: bitwise equal to the oracle's
    half-way stepper and to the single-part run, including the periodic
    wrap between the last and the first part (blocks)."""
    spec = lbm.GeometrySpec(kind, *dims)
    ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
    ref.load_perturbed(17)
    ref.advance(PARAMS, FORCE, 8)
    k = lbm.make_kernel(lbm.make_descriptor(name), spec, dist={"virtual_parts": parts})
    k.load_perturbed(17)
    k.advance(PARAMS, FORCE, 4)
    k.advance(PARAMS, FORCE, 4)
    assert np.array_equal(k.snapshot(), oracle_state(port, name, kind, dims, 8, 17))
    assert np.array_equal(k.snapshot(), ref.snapshot())
    assert abs(k.total_mass() - ref.total_mass()) <= 1e-12 * ref.total_mass()
    # macro fields and the fingerprint go through the per-part local arrays
    assert k.fingerprint() == ref.fingerprint()
    # the global adjacency is released after the local numbering is built
    with pytest.raises(lbm.ConfigError):
        k.export_structure()


def test_list_parts_nccl_transport_single_gpu(port):
    """The list halo over NCCL (pack -> grouped send/recv -> unpack on the comm
    stream), one NCCL rank owning every part (self send/recv)."""
    spec = lbm.GeometrySpec("blocks", 16, 16, 16)
    ref = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec)
    ref.load_perturbed(23)
    ref.advance(PARAMS, FORCE, 6)
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec,
                        dist={"virtual_parts": 3, "nccl_id": lbm.lbmgpu.nccl_unique_id()})
    k.load_perturbed(23)
    k.advance(PARAMS, FORCE, 6)
    assert np.array_equal(k.snapshot(), oracle_state(port, "list-aa-soa", "blocks", (16, 16, 16),
                                                     6, 23))
    assert np.array_equal(k.snapshot(), ref.snapshot())


def test_poiseuille_verification_passes():
    """verify_kernel (verification.cpp:31-100) on the GPU: slit 4x4x18."""
    for name in ("blk-push-soa", "aa-soa", "list-aa-soa", "list-pull-soa", "blk-pull-aos",
                 "list-push-aos"):
        r = lbm.verify_kernel(name, lbm.PoiseuilleCase(4, 4, 18, 1e-6, lbm.TrtParams.from_tau(0.9)))
        assert r["converged"] and r["passed"], (name, r["linf_rel"])
        assert r["linf_rel"] < 1e-6


@pytest.mark.parametrize("name", NAMES)
def test_poiseuille_every_kernel(name):
    """Reference acceptance criterion 6 (tests/acceptance.cpp:170-208) with its
    parameters: slit 8x8x34 (g=1e-6, interval 500, tol 3e-8) and 8x8x66
    (g=1e-6/4, interval 2000), 17/17 pass, L_inf not increasing above the
    1e-6 noise floor."""
    r34 = lbm.verify_kernel(name, lbm.PoiseuilleCase(8, 8, 34, 1e-6, lbm.TrtParams.from_tau(0.9)),
                            check_interval=500, rel_tol=3e-8, max_steps=100000)
    r66 = lbm.verify_kernel(name, lbm.PoiseuilleCase(8, 8, 66, 1e-6 / 4.0,
                                                     lbm.TrtParams.from_tau(0.9)),
                            check_interval=2000, rel_tol=3e-8, max_steps=200000)
    for r in (r34, r66):
        assert r["converged"] and r["passed"] and r["linf_rel"] < 1e-4, (name, r["linf_rel"])
    assert r66["linf_rel"] <= max(r34["linf_rel"], 1e-6)


def test_steady_state_reports_nonfinite():
    spec = lbm.GeometrySpec("channel", 8, 6, 6)
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), spec)
    s = k.snapshot()
    s[5] = np.nan
    k.load_state(s)
    with pytest.raises(lbm.NumericalError):
        k.steady_state_run(PARAMS, FORCE, 2, 1e-12, 10)


CONFIGS = os.path.join(os.path.dirname(__file__), "golden", "configs.json")


@pytest.mark.parametrize("cid", ["1", "2", "3", "4", "5"])
def test_baseline_config_fingerprint(cid):
    """BASELINE configs 1-4 at full size: default init, omega+ = 1,
    Lambda = 3/16, g = (1e-5, 0, 0); the final state's FNV-1a fingerprint
    must equal the reference's (made by tests/golden/make_golden.py)."""
    if not os.path.exists(CONFIGS):
        pytest.skip("configs.json not generated")
    gold = json.load(open(CONFIGS))
    if cid not in gold:
        pytest.skip(f"config {cid} golden not generated")
    c = gold[cid]
    spec = lbm.GeometrySpec(c["kind"], *c["dims"], c.get("block", 4), c.get("spacing", 4),
                            c.get("pipe_diameter", 0))
    k = lbm.make_kernel(lbm.make_descriptor(c["kernel"]), spec)
    assert k.n_fluid() == c["n_fluid"]
    if c["kernel"].startswith("list-"):
        _, _, starts, total = k.export_structure()
        assert [int(v) for v in starts] == c["starts_auto"]
        assert total == c["total_slots_auto"]
    m0 = k.total_mass()
    assert abs(m0 - c["mass0"]) <= 1e-12 * c["mass0"]
    k.advance(lbm.TrtParams(1.0, 3.0 / 16.0), lbm.BodyForce(tuple(c["g"])), c["steps"])
    assert f"{k.fingerprint():016x}" == c["fingerprint"]
    assert abs(k.total_mass() - c["mass1"]) <= 1e-12 * c["mass1"]


@pytest.mark.parametrize("cid", ["2", "3", "4"])
def test_baseline_config_structure_bitwise(cid, port):
    """north_star: node lists and adjacency bit-exact at full size.  For the
    list configs the device-built structure is exported (canonical order:
    nodes as int32 (x, y, z), adjacency adj[n*18 + d-1] as u32) and its
    FNV-1a must equal the reference's build_structure (list_lattice.cpp:
    149-204; goldens from tests/golden/make_golden.py) for both orientations
    (Gather: list-pull-soa, Scatter: list-aa-soa) and both paddings (auto,
    none), together with the 19 start offsets and the slot total."""
    if not os.path.exists(CONFIGS):
        pytest.skip("configs.json not generated")
    gold = json.load(open(CONFIGS))
    c = gold[cid]
    spec = lbm.GeometrySpec(c["kind"], *c["dims"], c.get("block", 4), c.get("spacing", 4),
                            c.get("pipe_diameter", 0))
    for pad, policy in (("auto", lbm.PaddingPolicy.automatic()), ("none", lbm.PaddingPolicy.none())):
        for orient, name in (("gather", "list-pull-soa"), ("scatter", "list-aa-soa")):
            k = lbm.make_kernel(lbm.make_descriptor(name), spec, policy)
            nodes, adj, starts, total = k.export_structure()
            k.close()
            del k
            assert [int(v) for v in starts] == c[f"starts_{pad}"], (pad, orient)
            assert total == c[f"total_slots_{pad}"], (pad, orient)
            assert f"{port.fingerprint(adj):016x}" == c[f"adj_fnv_{pad}_{orient}"], (pad, orient)
            if pad == "auto" and orient == "gather":
                nv = np.ascontiguousarray(nodes, np.int32).view(np.uint32).ravel()
                assert f"{port.fingerprint(nv):016x}" == c["nodes_fnv"]
            del nodes, adj


@pytest.mark.parametrize("cid,variant", [("2", "ria"), ("4", "ria"), ("5", "peer8"),
                                         ("2", "ranges4"),
                                         pytest.param("5", "copy4", marks=pytest.mark.slow)])
def test_baseline_config_fingerprint_alternative_paths(cid, variant, monkeypatch):
    """The BASELINE golden fingerprints at full size through the other paths:
    list-aa-ria-soa (cfg 2: 8-bit pattern ids, cfg 4: 32-bit ids), cfg 5 as
    8 emulated z slabs over the peer transport (boundary stream, flags) and
    as 4 slabs over device-copy halos (marked slow: ~50 s), and cfg 2 as 4
    emulated node ranges (list-aa-soa node-range decomposition, index-list
    halos; reference kernels_list_aa.cpp:63-74 splits the same contiguous
    node ranges over its workers)."""
    if not os.path.exists(CONFIGS):
        pytest.skip("configs.json not generated")
    gold = json.load(open(CONFIGS))
    if cid not in gold:
        pytest.skip(f"config {cid} golden not generated")
    c = gold[cid]
    spec = lbm.GeometrySpec(c["kind"], *c["dims"], c.get("block", 4), c.get("spacing", 4),
                            c.get("pipe_diameter", 0))
    name, dist = c["kernel"], None
    if variant == "ria":
        name = "list-aa-ria-soa"
    elif variant == "peer8":
        dist = {"virtual_parts": 8, "transport": "peer"}
    elif variant == "copy4":
        dist = {"virtual_parts": 4}
    elif variant == "ranges4":
        dist = {"virtual_parts": 4}
    k = lbm.make_kernel(lbm.make_descriptor(name), spec, dist=dist)
    k.kernel_stats_enable(True)
    k.advance(lbm.TrtParams(1.0, 3.0 / 16.0), lbm.BodyForce(tuple(c["g"])), c["steps"])
    assert f"{k.fingerprint():016x}" == c["fingerprint"], (cid, variant)
    assert abs(k.total_mass() - c["mass1"]) <= 1e-12 * c["mass1"]
    names = set(k.kernel_stats())
    expect = {"ria": "list_aa_odd_ria_pid", "peer8": "full_aa_odd_soa_peer",
              "copy4": "full_aa_odd_soa_halo", "ranges4": "list_aa_odd"}[variant]
    assert any(n.startswith(expect) for n in names), names


def test_custom_flagfield_path(port):
    """make_kernel takes any FlagField (kernels.hpp:102-105): a host flag
    field uploaded through LBMGPU_CUSTOM gives the same results as the device
    generator, and an irregular hand-made geometry matches the oracle."""
    spec = lbm.GeometrySpec("pipe", 9, 12, 13)
    ff = lbm.build_geometry(spec)
    fl, per, nf = port.geometry("pipe", 9, 12, 13)
    assert np.array_equal(ff.flags, fl) and ff.periodic == tuple(bool(p) for p in per)
    for name in ("aa-soa", "list-pull-soa", "blk-push-aos"):
        a = lbm.make_kernel(lbm.make_descriptor(name), spec)
        b = lbm.make_kernel(lbm.make_descriptor(name), ff)
        for k in (a, b):
            k.load_perturbed(3)
            k.advance(PARAMS, FORCE, 6)
        assert np.array_equal(a.snapshot(), b.snapshot()), name
    # random obstacles inside a fully periodic box: compare to the oracle's
    # half-way stepper through the reference neighbor rule
    rng = np.random.default_rng(5)
    flags = (rng.random(10 * 9 * 8) < 0.2).astype(np.uint8)
    custom = lbm.FlagField(10, 9, 8, (True, True, True), flags)
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), custom)
    nfl = int(np.count_nonzero(flags == 0))
    assert k.n_fluid() == nfl
    k.load_perturbed(11)
    k.advance(PARAMS, FORCE, 4)
    got = k.snapshot()
    # oracle on the same flags: reuse the C stepper through a blocks spec is
    # impossible, so compare against a direct per-node restatement
    init = lbm.perturbed_equilibrium(nfl, 11)
    expect = _halfway_reference(port, flags, (10, 9, 8), init, 4)
    assert np.array_equal(got, expect)


def _halfway_reference(port, flags, dims, init, steps):
    """Half-way bounce-back textbook stepper (tests/support/reference.hpp:72-105)
    in numpy + the oracle collision, fully periodic."""
    nx, ny, nz = dims
    cxs = [0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0]
    cys = [0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1]
    czs = [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1]
    opp = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
    solid = flags.reshape(nx, ny, nz)
    fluid = [(x, y, z) for x in range(nx) for y in range(ny) for z in range(nz) if not solid[x, y, z]]
    f = {c: init[i * 19:(i + 1) * 19].copy() for i, c in enumerate(fluid)}
    wp, wm = PARAMS.omega_plus, port.omega_minus(PARAMS.omega_plus)
    for _ in range(steps):
        post = {c: port.collide(v, wp, wm, G_TEST) for c, v in f.items()}
        nxt = {}
        for (x, y, z) in fluid:
            q = np.empty(19)
            q[0] = post[(x, y, z)][0]
            for d in range(1, 19):
                s = ((x - cxs[d]) % nx, (y - cys[d]) % ny, (z - czs[d]) % nz)
                q[d] = post[s][d] if not solid[s] else post[(x, y, z)][opp[d]]
            nxt[(x, y, z)] = q
        f = nxt
    return np.concatenate([f[c] for c in fluid])


def test_local_rows_round_trip_on_split_domain():
    """Process-local row access (the multi-process e2e path) on an emulated
    3-slab split: rows are the slabs' fluid nodes in canonical order."""
    spec = lbm.GeometrySpec("channel", 16, 12, 24)
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), spec, dist={"virtual_parts": 3})
    k.load_perturbed(7)
    k.advance(PARAMS, FORCE, 4)
    full = k.snapshot().reshape(-1, 19)
    idx = k.local_canonical_index()
    assert k.local_rows() == k.n_fluid() and np.array_equal(np.sort(idx), np.arange(k.n_fluid()))
    loc = k.snapshot_local().reshape(-1, 19)
    assert np.array_equal(full[idx], loc)
    k.load_state_local(np.zeros(loc.size))
    assert np.count_nonzero(k.snapshot()) == 0
    k.load_state_local(loc.reshape(-1))
    assert np.array_equal(k.snapshot().reshape(-1, 19), full)


@pytest.mark.parametrize("case", range(32))
def test_randomized_against_oracle(case, port, monkeypatch):
    """Seeded random cases against the oracle's textbook steppers: random
    geometry kind and box (often a multiple of 16 in x, so the AoS halo
    tiles and the 128-node AA blocks see ragged y/z), kernel name, blk,
    relaxation time, body force, step count and launch path (fused or
    per-sweep); bitwise."""
    rng = np.random.default_rng(7000 + case)
    while True:
        kind = str(rng.choice(["channel", "slit", "pipe", "blocks"]))
        nx = int(rng.choice([16, 32, 48])) if rng.random() < 0.5 else int(rng.integers(1, 30))
        ny, nz = int(rng.integers(3, 22)), int(rng.integers(3, 22))
        block, spacing = int(rng.integers(1, 5)), int(rng.integers(0, 4))
        try:
            _, _, nf = port.geometry(kind, nx, ny, nz, block, spacing)
        except ValueError:
            continue
        if nf > 0:
            break
    name = str(rng.choice(NAMES))
    blk = int(rng.integers(0, 4)) if name.startswith("list-") else 0
    tau = float(rng.uniform(0.55, 1.9))
    g = tuple(float(v) for v in rng.uniform(-2e-5, 2e-5, 3))
    steps = int(rng.integers(1, 5)) * 2 if "aa" in name.split("-") else int(rng.integers(1, 9))
    monkeypatch.setenv("LBMGPU_FUSED_MB", str(rng.choice(["96", "0"])))
    init = port.perturbed(nf, 100 + case)
    fam = "half" if name.startswith("list-") else "full"
    params = lbm.TrtParams.from_tau(tau)
    expect, mass = port.run(fam, kind, nx, ny, nz, steps, params.omega_plus, g=g, init=init,
                            block=block, spacing=spacing)
    k = lbm.make_kernel(lbm.make_descriptor(name, blk=blk),
                        lbm.GeometrySpec(kind, nx, ny, nz, block, spacing))
    k.load_state(init)
    k.advance(params, lbm.BodyForce(g), steps)
    got = k.snapshot()
    assert np.array_equal(got, expect), (name, kind, (nx, ny, nz), blk, tau, steps)


def test_snapshot_out_buffer_validation():
    """snapshot(out=...) / snapshot_local(out=...) write N*19 doubles at the
    array's data pointer: float32, strided or wrongly sized arrays are
    rejected before the C ABI is called."""
    k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("blocks", 12, 10, 10))
    n = k.n_fluid() * 19
    for bad in (np.empty(n, np.float32), np.empty(2 * n)[::2], np.empty(n - 1),
                np.empty(n + 19), np.empty(n, np.int64)):
        with pytest.raises(ValueError):
            k.snapshot(out=bad)
        with pytest.raises(ValueError):
            k.snapshot_local(out=bad)
    good = np.empty(n)
    assert k.snapshot(out=good) is good and np.array_equal(good, k.snapshot())


@pytest.mark.parametrize("name,dist", [
    ("aa-soa", {"virtual_parts": 8, "transport": "peer"}),
    ("aa-soa", {"virtual_parts": 8}),
    ("blk-pull-soa", {"virtual_parts": 4, "transport": "peer"}),
    ("list-aa-soa", {"virtual_parts": 4})])
def test_boundary_stream_overlaps_interior(name, dist):
    """Overlap evidence for the decomposed paths (SURVEY 8(e) schedule): the
    per-launch device intervals (kernel timeline, events on both streams)
    show the boundary-stream work -- boundary sweeps, peer waits / signals,
    halo exchanges -- running while interior sweeps run.  Emulated slabs /
    node ranges on one GPU (channel 512x128x128)."""
    k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec("channel", 512, 128, 128),
                        dist=dist)
    k.advance(PARAMS, FORCE, 2)
    k.synchronize()
    k.kernel_stats_reset()
    k.kernel_stats_enable(True)
    k.advance(PARAMS, FORCE, 8)
    k.kernel_stats_enable(False)
    tl = k.kernel_timeline()
    assert len(tl) > 0
    ov = lbm.lbmgpu.stream_overlap(tl)
    assert ov["boundary_ms"] > 0, tl[:10]
    assert ov["frac"] > 0.5, ov

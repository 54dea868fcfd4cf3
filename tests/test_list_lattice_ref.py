"""The reference's list-lattice tests (proj/tests/test_list_lattice.cpp), case by
case, against the device structure builder (k_build_adj / the node scan,
exported through lbmgpu_export_structure), the padding rules and the run
coding statistics.

The kernel name picks what the reference passes to build_structure: the
list-pull names build the Gather table, list-push / list-aa the Scatter
table, the -aos names the AoS slot map; the run coding comes back through
lbmgpu_export_runs / lbmgpu_vectorizable_fraction.  Not mirrored: the
layer-condition bound (a CPU cache model, test_list_lattice.cpp:72-78).
"""
import numpy as np
import pytest

import paper_1711_11468_b200 as lbm

gpu = pytest.mark.gpu

C = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
     (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 0, 1), (-1, 0, -1), (1, 0, -1),
     (-1, 0, 1), (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1)]
OPP = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
W = [1 / 3] + [1 / 18] * 6 + [1 / 36] * 12


def all_fluid(nx, ny, nz):
    return lbm.FlagField(nx, ny, nz, (True, True, True), np.zeros(nx * ny * nz, np.uint8))


def flagfield(geom):
    return geom if isinstance(geom, lbm.FlagField) else lbm.build_geometry(geom)


class Structure:
    """ListStructure (list_lattice.hpp:66-99) as the device built it."""

    def __init__(self, name, geom, blk=0, pad=None):
        self.k = lbm.make_kernel(lbm.make_descriptor(name, blk), geom, pad or lbm.PaddingPolicy.none())
        nodes, adj, starts, self.total = self.k.export_structure()
        self.nodes = [tuple(int(v) for v in c) for c in nodes]
        self.adj = adj.reshape(-1, 18)
        self.starts = [int(s) for s in starts]
        self.rank = {c: n for n, c in enumerate(self.nodes)}
        self.gather = "pull" in name
        self.soa = name.endswith("soa")
        self.ff = flagfield(geom)

    def slot(self, n, d):  # SlotMap::slot
        return self.starts[d] + n if self.soa else 19 * n + d

    def entry(self, n, d):
        return int(self.adj[n, d - 1])

    def neighbor(self, c, d):
        """geometry.cpp:119-131: wrap on periodic axes, else outside; None for
        outside or a solid hit, else the fluid coordinate."""
        p = [c[0] + C[d][0], c[1] + C[d][1], c[2] + C[d][2]]
        for a, n in enumerate((self.ff.nx, self.ff.ny, self.ff.nz)):
            if p[a] < 0 or p[a] >= n:
                if not self.ff.periodic[a]:
                    return None
                p[a] %= n
        return tuple(p) if self.ff.flags[self.ff.index(*p)] == 0 else None

    def walk_entry(self, n, d):  # test_list_lattice.cpp:24-31
        nb = self.neighbor(self.nodes[n], OPP[d] if self.gather else d)
        return self.slot(self.rank[nb], d) if nb is not None else self.slot(n, OPP[d])

    def check_walk(self):
        for n in range(len(self.nodes)):
            for d in range(1, 19):
                assert self.entry(n, d) == self.walk_entry(n, d), (n, d)


# ---- order_nodes ---------------------------------------------------------------
@gpu
def test_order_nodes_blk0_is_the_plain_xyz_nest():
    """test_list_lattice.cpp:35-42."""
    s = Structure("list-aa-soa", all_fluid(2, 2, 2))
    assert s.nodes == [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 0), (1, 0, 1), (1, 1, 0),
                       (1, 1, 1)]


@gpu
def test_order_nodes_on_the_channel_keeps_z_lines_consecutive():
    """test_list_lattice.cpp:44-56."""
    s = Structure("list-aa-soa", lbm.GeometrySpec("channel", 6, 8, 8))
    assert len(s.nodes) == 6 * 6 * 6
    for n in range(len(s.nodes)):
        if n % 6 > 0:
            (x, y, z), (px, py, pz) = s.nodes[n], s.nodes[n - 1]
            assert (x, y, z) == (px, py, pz + 1)


@gpu
def test_order_nodes_blk_tiles_the_yz_plane():
    """test_list_lattice.cpp:58-70: first tile (ty, tz) = (0, 0), x = 0 then 1."""
    s = Structure("list-aa-soa", all_fluid(2, 4, 4), blk=2)
    assert len(s.nodes) == 32 and len(set(s.nodes)) == 32
    assert s.nodes[:8] == [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 0), (1, 0, 1),
                           (1, 1, 0), (1, 1, 1)]


# ---- adjacency -----------------------------------------------------------------
@gpu
def test_single_fluid_node_closes_onto_itself():
    """test_list_lattice.cpp:80-91."""
    flags = np.ones(27, np.uint8)
    flags[(1 * 3 + 1) * 3 + 1] = 0
    ff = lbm.FlagField(3, 3, 3, (True, True, True), flags)
    for name in ("list-pull-soa", "list-push-soa"):  # Gather, Scatter
        s = Structure(name, ff)
        assert len(s.nodes) == 1
        for d in range(1, 19):
            assert s.entry(0, d) == s.slot(0, OPP[d])


@gpu
def test_fully_periodic_all_fluid_adjacency_matches_the_geometry_walk():
    """test_list_lattice.cpp:93-103: both orientations, both layouts."""
    for name in ("list-pull-soa", "list-pull-aos", "list-push-soa", "list-push-aos"):
        Structure(name, all_fluid(4, 4, 4)).check_walk()


@gpu
def test_adjacency_walk_oracle_on_mixed_geometries_both_orientations():
    """test_list_lattice.cpp:105-118: blocks 8^3 (b = s = 2) and slit 6x6x8,
    blk 0 and 2, padding auto."""
    for geom in (lbm.GeometrySpec("blocks", 8, 8, 8, 2, 2), lbm.GeometrySpec("slit", 6, 6, 8)):
        for name in ("list-pull-soa", "list-aa-soa"):
            for blk in (0, 2):
                Structure(name, geom, blk, lbm.PaddingPolicy.automatic()).check_walk()


@gpu
def test_gather_and_scatter_tables_are_mutually_consistent():
    """test_list_lattice.cpp:120-143."""
    geom = lbm.GeometrySpec("blocks", 8, 6, 6, 2, 2)
    gather, scatter = Structure("list-pull-soa", geom), Structure("list-push-soa", geom)
    assert gather.nodes == scatter.nodes
    for n, c in enumerate(gather.nodes):
        for d in range(1, 19):
            nb = gather.neighbor(c, d)
            if nb is not None:
                m = gather.rank[nb]
                assert scatter.entry(n, d) == gather.slot(m, d)
                assert gather.entry(m, d) == gather.slot(n, d)
            else:
                assert scatter.entry(n, d) == gather.slot(n, OPP[d])


# ---- padding (host rules, no device call) -----------------------------------------
def cache_set_of(elem):  # list_lattice.cpp:52-54: 64-byte lines, 512 sets
    return elem * 8 // 64 % 512


def tlb_set_of(elem):  # list_lattice.cpp:56-58: 2 MiB pages, 4 sets
    return elem * 8 // (2 << 20) % 4


def test_padding_offsets_none():
    """test_list_lattice.cpp:145-148."""
    starts, _ = lbm.padding_offsets(1000, lbm.PaddingPolicy.none())
    assert [int(s) for s in starts] == [1000 * d for d in range(19)]


def test_padding_offsets_auto_spreads_cache_and_tlb_sets():
    """test_list_lattice.cpp:150-164."""
    for n in (27, 1000, 100000):
        starts, total = lbm.padding_offsets(n, lbm.PaddingPolicy.automatic())
        starts = [int(s) for s in starts]
        for d in range(19):
            assert starts[d] >= (0 if d == 0 else starts[d - 1] + n)
            assert cache_set_of(starts[d]) == (512 // 19) * d % 512
            assert tlb_set_of(starts[d]) == d % 4
        assert len({cache_set_of(s) for s in starts}) == 19
        assert total >= starts[18] + n


def test_padding_offsets_thrash_maps_every_start_to_one_set():
    """test_list_lattice.cpp:166-173."""
    starts, _ = lbm.padding_offsets(5000, lbm.PaddingPolicy.thrash())
    starts = [int(s) for s in starts]
    for d in range(19):
        assert cache_set_of(starts[d]) == cache_set_of(starts[0])
        assert tlb_set_of(starts[d]) == tlb_set_of(starts[0])
        if d > 0:
            assert starts[d] >= starts[d - 1] + 5000


def test_padding_policy_parsing():
    """test_list_lattice.cpp:175-190."""
    for mode in ("auto", "none", "thrash"):
        assert lbm.PaddingPolicy.parse(mode).mode == mode
    p = lbm.PaddingPolicy.parse(",".join(str(i) for i in range(1, 20)))
    assert p.mode == "explicit" and p.pads[0] == 1 and p.pads[18] == 19
    starts, _ = lbm.padding_offsets(10, p)
    assert int(starts[0]) == 1 and int(starts[1]) == 1 + 10 + 2
    assert lbm.PaddingPolicy.parse(p.to_string()).pads == p.pads
    for bad in ("1,2,3", "bogus"):
        with pytest.raises(lbm.ConfigError):
            lbm.PaddingPolicy.parse(bad)


# ---- run coding -------------------------------------------------------------------
class Coding:
    """RiaCoding (list_lattice.hpp:52-64) of a run-coded kernel: run starts
    and lengths from the device builder."""

    def __init__(self, geom, blk=0, pad=None):
        self.s = Structure("list-aa-ria-soa", geom, blk, pad)
        self.k = self.s.k
        self.n_fluid = self.k.n_fluid()
        self.start = [int(v) for v in self.k.export_runs()]
        self.length = [b - a for a, b in zip(self.start, self.start[1:] + [self.n_fluid])]

    def total_runs(self):
        return len(self.start)

    def v(self, w):
        return self.k.vectorizable_fraction(w)


@gpu
def test_ria_on_a_small_channel_runs_of_1_interior_1_per_z_line():
    """test_list_lattice.cpp:192-209: 20 * 8 z lines of 8 fluid nodes, each
    split (1, 6, 1): v(W=4) = 4/8, v(W=1) = 1."""
    ria = Coding(lbm.GeometrySpec("channel", 20, 10, 10))
    assert ria.total_runs() == 3 * 20 * 8
    assert ria.k.ria_stats() == {"total_runs": 3 * 20 * 8, "n_fluid": 20 * 8 * 8}
    assert ria.length == [1, 6, 1] * (20 * 8)
    assert ria.v(4) == pytest.approx(4.0 / 8.0)
    assert ria.v(1) == 1.0
    assert ria.k.vector_fraction() == ria.v(4)  # the descriptor's W = 4


@gpu
def test_ria_losslessness_expanding_runs_reproduces_the_adjacency():
    """test_list_lattice.cpp:211-234: inside a run every node's entries sit
    at the same offsets from its own slots (the run's pattern), so run
    starts + one pattern per run reproduce the table; the runs cover every
    node once."""
    for geom in (lbm.GeometrySpec("blocks", 8, 8, 8, 2, 2), lbm.GeometrySpec("channel", 12, 8, 8)):
        for blk in (0, 2):
            for pad in (lbm.PaddingPolicy.none(), lbm.PaddingPolicy.automatic()):
                ria = Coding(geom, blk, pad)
                s = ria.s
                own = np.array([[s.slot(n, d) for d in range(1, 19)]
                                for n in range(ria.n_fluid)], np.int64)
                rel = s.adj.astype(np.int64) - own
                for start, length in zip(ria.start, ria.length):
                    assert length >= 1
                    assert np.all(rel[start:start + length] == rel[start])
                assert sum(ria.length) == ria.n_fluid
                # runs are maximal: the pattern changes at every run start
                for start in ria.start[1:]:
                    assert np.any(rel[start] != rel[start - 1])


@gpu
def test_blocking_factor_2_kills_vectorizability():
    """test_list_lattice.cpp:236-244."""
    ria = Coding(lbm.GeometrySpec("channel", 20, 10, 10), blk=2)
    assert max(ria.length) <= 2
    assert ria.v(4) == 0.0


@gpu
def test_isolated_patterns_give_all_length_1_runs():
    """test_list_lattice.cpp:246-256."""
    ria = Coding(lbm.GeometrySpec("blocks", 6, 6, 6, 1, 1))
    assert ria.total_runs() == ria.n_fluid and set(ria.length) == {1}


@gpu
def test_v_is_non_increasing_along_divisibility_chains_of_w():
    """test_list_lattice.cpp:258-277."""
    geom = lbm.GeometrySpec("blocks", 12, 9, 9, 3, 3)
    for blk in (0, 3):
        ria = Coding(geom, blk)
        prev = 1.0
        for w in (1, 2, 4, 8, 16, 32):
            assert ria.v(w) <= prev + 1e-15
            prev = ria.v(w)
        for w in (3, 5, 7):
            for k in (2, 3, 4):
                assert ria.v(k * w) <= ria.v(w) + 1e-15
        assert ria.v(1) == 1.0
        # the library's count equals the definition over the exported runs
        for w in (2, 3, 8):
            assert ria.v(w) == sum(n // w * w for n in ria.length) / ria.n_fluid


@gpu
def test_padding_does_not_change_the_run_structure():
    """test_list_lattice.cpp:279-299."""
    geom = lbm.GeometrySpec("channel", 12, 8, 8)
    base = Coding(geom, pad=lbm.PaddingPolicy.none())
    for pad in (lbm.PaddingPolicy.automatic(), lbm.PaddingPolicy.thrash()):
        ria = Coding(geom, pad=pad)
        assert (ria.start, ria.length) == (base.start, base.length)


@gpu
def test_run_export_only_for_run_coded_names():
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("channel", 6, 8, 8))
    assert k.export_runs() is None and k.vectorizable_fraction(4) is None
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-pv-soa"), lbm.GeometrySpec("channel", 6, 8, 8))
    with pytest.raises(lbm.ConfigError, match="W must be >= 1"):
        k.vectorizable_fraction(0)


# ---- the lattice ------------------------------------------------------------------
@gpu
def test_list_lattice_init_snapshot_mass():
    """test_list_lattice.cpp:301-319."""
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("blocks", 8, 8, 8, 2, 2))
    snap = k.snapshot()
    assert snap.size == k.n_fluid() * 19
    assert np.array_equal(snap.reshape(-1, 19), np.tile(W, (k.n_fluid(), 1)))
    assert k.total_mass() == pytest.approx(float(k.n_fluid()), rel=1e-12)
    state = np.random.default_rng(9).uniform(0.01, 1.0, snap.size)
    k.load_state(state)
    assert np.array_equal(k.snapshot(), state)

"""The reference's geometry tests (proj/tests/test_geometry.cpp), case by case,
against the device generator (lbmgpu_geometry_build -> k_flags + census) and
the `neighbor` rule as the device structure builder applies it
(lbmgpu_export_structure)."""
import math

import numpy as np
import pytest

import paper_1711_11468_b200 as lbm

gpu = pytest.mark.gpu


def grid(ff):
    """flags as [x, y, z] (FlagField order (x*ny + y)*nz + z)."""
    return np.asarray(ff.flags).reshape(ff.nx, ff.ny, ff.nz)


@gpu
def test_channel_census():
    """test_geometry.cpp:10-14."""
    ff = lbm.build_geometry(lbm.GeometrySpec("channel", 500, 100, 100))
    assert lbm.fluid_count(ff) == 4802000
    assert tuple(ff.periodic) == (True, False, False)


@gpu
def test_channel_fluid_count_formula():
    """test_geometry.cpp:16-25: 20 random boxes, nx * (ny-2) * (nz-2)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        nx, ny, nz = (int(v) for v in rng.integers(3, 25, 3))
        ff = lbm.build_geometry(lbm.GeometrySpec("channel", nx, ny, nz))
        assert lbm.fluid_count(ff) == nx * (ny - 2) * (nz - 2), (nx, ny, nz)


@gpu
def test_slit_walls_sit_at_the_z_extremes_only():
    """test_geometry.cpp:27-37."""
    ff = lbm.build_geometry(lbm.GeometrySpec("slit", 8, 8, 10))
    assert lbm.fluid_count(ff) == 8 * 8 * 8
    assert tuple(ff.periodic) == (True, True, False)
    g = grid(ff)
    assert np.all(g[:, :, 0] != 0) and np.all(g[:, :, 9] != 0) and np.all(g[:, :, 1:9] == 0)


@gpu
def test_blocks_census_against_an_enumeration_oracle():
    """test_geometry.cpp:39-63."""
    ff = lbm.build_geometry(lbm.GeometrySpec("blocks", 16, 16, 16, 4, 4))
    assert lbm.fluid_count(ff) == 16 ** 3 - 8 * 4 ** 3  # 3584
    oracle = 0
    for x in range(16):
        for y in range(16):
            for z in range(16):
                inside = any(bx <= x < bx + 4 and by <= y < by + 4 and bz <= z < bz + 4
                             for bx in (4, 12) for by in (4, 12) for bz in (4, 12))
                oracle += not inside
    assert lbm.fluid_count(ff) == oracle
    assert tuple(ff.periodic) == (True, True, True)
    g = grid(ff)
    assert g[0, 0, 0] == 0 and g[4, 4, 4] != 0  # obstacles start after `spacing` fluid layers


@gpu
def test_blocks_fluid_fraction_is_exact_on_period_multiples():
    """test_geometry.cpp:65-78."""
    for b in (1, 2, 3):
        for s in (1, 2, 4):
            n = 2 * (b + s)
            ff = lbm.build_geometry(lbm.GeometrySpec("blocks", n, n, n, b, s))
            assert lbm.fluid_count(ff) / ff.volume() == pytest.approx(1.0 - (b / (b + s)) ** 3,
                                                                      rel=1e-12)


def test_fluid_count_on_an_all_fluid_field():
    """test_geometry.cpp:80-85 (host function)."""
    ff = lbm.FlagField(4, 4, 4, (True, True, True), np.zeros(64, np.uint8))
    assert lbm.fluid_count(ff) == 64


@gpu
def test_neighbor_periodic_wrap_and_solid_hits():
    """test_geometry.cpp:87-104 through the Scatter adjacency the device
    builder writes (list_lattice.cpp:177-191): a fluid neighbour m gives
    slot(rank[m], d), a solid hit gives the own slot(n, opp d); with padding
    none slot(n, d) = d * N + n.  W = 2, N = 3, S = 4."""
    def structure(spec):
        k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec, lbm.PaddingPolicy.none())
        nodes, adj, starts, _ = k.export_structure()
        rank = {tuple(int(v) for v in c): n for n, c in enumerate(nodes)}
        return adj.reshape(-1, 18), [int(s) for s in starts], rank

    adj, starts, rank = structure(lbm.GeometrySpec("channel", 12, 8, 8))
    n = rank[(0, 5, 5)]
    assert adj[n, 2 - 1] == starts[2] + rank[(11, 5, 5)]  # wraps along periodic x
    n = rank[(3, 1, 5)]
    assert adj[n, 4 - 1] == starts[3] + n  # y = 0 is a wall: bounce back into opp(S) = N
    adj, starts, rank = structure(lbm.GeometrySpec("slit", 4, 4, 6))
    n = rank[(0, 3, 2)]
    assert adj[n, 3 - 1] == starts[3] + rank[(0, 0, 2)]  # the slit is periodic in y
    # the boundary layer z = 0 is solid, so no fluid node ever looks outside the box
    assert all(1 <= z <= 4 for (_, _, z) in rank)


@gpu
def test_pipe_staircase_fraction_approximates_the_circle_area():
    """test_geometry.cpp:106-120."""
    ff = lbm.build_geometry(lbm.GeometrySpec("pipe", 20, 21, 21))
    r = (21 - 2) / 2.0
    circle = math.pi * r * r / (21.0 * 21.0)
    got = lbm.fluid_count(ff) / ff.volume()
    assert abs(got - circle) / circle < 0.15
    disc = sum(1 for y in range(21) for z in range(21)
               if (y - 10.0) ** 2 + (z - 10.0) ** 2 <= r * r)
    assert lbm.fluid_count(ff) == disc * 20


@gpu
def test_geometry_generation_is_deterministic():
    """test_geometry.cpp:122-127."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10, 3, 2)
    assert np.array_equal(lbm.build_geometry(spec).flags, lbm.build_geometry(spec).flags)


@gpu
def test_flags_are_invariant_along_periodic_axes():
    """test_geometry.cpp:129-141."""
    for spec in (lbm.GeometrySpec("channel", 6, 7, 8), lbm.GeometrySpec("pipe", 5, 9, 9)):
        g = grid(lbm.build_geometry(spec)) != 0
        assert np.all(g == g[0])


def test_configuration_errors_before_device_work():
    """test_geometry.cpp:143-155: dimension and obstacle checks are host-side
    (no GPU needed); an unknown kind lists the valid ones."""
    for spec in (("channel", 4, 2, 5), ("slit", 4, 4, 2), ("pipe", 4, 3, 3), ("blocks", 4, 4, 4, 5, 1)):
        with pytest.raises(lbm.ConfigError):
            lbm.build_geometry(lbm.GeometrySpec(*spec))
    with pytest.raises(lbm.ConfigError, match="valid: channel, slit, pipe, blocks"):
        lbm.build_geometry(lbm.GeometrySpec("torus", 4, 4, 4))


@gpu
def test_no_fluid_at_all_is_a_configuration_error():
    """test_geometry.cpp:151-153: blocks with spacing 0 leave no fluid node
    (the device census finds it)."""
    with pytest.raises(lbm.ConfigError, match="no fluid"):
        lbm.build_geometry(lbm.GeometrySpec("blocks", 4, 4, 4, 2, 0))

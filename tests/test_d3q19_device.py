"""The reference's model tests (proj/tests/test_d3q19.cpp) for the collision,
run on the device: one blk-push step over a fully periodic all-fluid box
writes f*_i(x) to x + c_i, so un-streaming the snapshot on the host gives the
device's post-collision PDFs of every node -- 1,000 nodes = the reference's
1,000 random trials.  The same states go through the oracle's collide_node,
which the device result must equal bit for bit.

Host-side cases (stencil identities, TrtParams relations) use the Python
mirror's tables; the equilibrium used as test input is restated here from
d3q19.cpp (f_i = w_i rho (1 + 3 cu + 4.5 cu^2 - 1.5 u^2)).
"""
import numpy as np
import pytest

import paper_1711_11468_b200 as lbm

gpu = pytest.mark.gpu

C = np.array([(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
              (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 0, 1), (-1, 0, -1), (1, 0, -1),
              (-1, 0, 1), (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1)])
OPP = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
N = 10  # 10^3 nodes


def random_states(seed):
    """random_state (test_d3q19.cpp:12-17): f_i = w_i * U(0.5, 1.5), 1,000 nodes."""
    return W * np.random.default_rng(seed).uniform(0.5, 1.5, size=(N ** 3, 19))


def equilibrium(rho, u):
    cu = C @ np.asarray(u, float)
    return W * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * float(np.dot(u, u)))


def device_collide(f, params, g):
    """Post-collision PDFs of every node, collided by the device's push sweep."""
    box = lbm.FlagField(N, N, N, (True, True, True), np.zeros(N ** 3, np.uint8))
    k = lbm.make_kernel(lbm.make_descriptor("blk-push-soa"), box)
    k.load_state(np.ascontiguousarray(f).reshape(-1))
    k.advance(params, lbm.BodyForce(tuple(g)), 1)
    after = k.snapshot().reshape(N, N, N, 19)
    post = np.empty_like(after)
    for i in range(19):  # f*_i(x) = after_i(x + c_i)
        post[..., i] = np.roll(after[..., i], shift=tuple(-C[i]), axis=(0, 1, 2))
    return post.reshape(-1, 19)


# ---- host tables ---------------------------------------------------------------
def test_stencil_constants_exact_integer_moment_identities():
    """test_d3q19.cpp:21-55 on the tables the tests and the host mirror share;
    the device's copies are pinned by every parity test."""
    assert tuple(C[0]) == (0, 0, 0)
    assert all(int(np.dot(C[i], C[i])) == 1 and W[i] == 1.0 / 18.0 for i in range(1, 7))
    assert all(int(np.dot(C[i], C[i])) == 2 and W[i] == 1.0 / 36.0 for i in range(7, 19))
    assert W[0] == 1.0 / 3.0
    w36 = np.array([12] + [2] * 6 + [1] * 12)
    assert np.allclose(w36, W * 36, rtol=1e-15)
    assert w36.sum() == 36 and np.all(w36 @ C == 0)
    assert np.array_equal(np.einsum("i,ia,ib->ab", w36, C, C), 12 * np.eye(3, dtype=int))


def test_opp_is_an_involution_with_c_opp_equal_minus_c():
    """test_d3q19.cpp:57-63."""
    for i in range(19):
        assert OPP[OPP[i]] == i and np.array_equal(C[OPP[i]], -C[i]) and W[OPP[i]] == W[i]


def test_trt_params_relations():
    """test_d3q19.cpp:65-72."""
    p = lbm.TrtParams.from_tau(0.9)
    assert p.viscosity() == pytest.approx(2.0 / 15.0, rel=1e-15)
    lhs = (1.0 / p.omega_plus - 0.5) * (1.0 / p.omega_minus() - 0.5)
    assert lhs == pytest.approx(3.0 / 16.0, rel=1e-14)
    for bad in (0.0, 2.0):
        with pytest.raises(lbm.ConfigError):
            lbm.TrtParams(bad).validate()


# ---- the collision on the device ------------------------------------------------
@gpu
def test_trt_collide_equilibrium_is_a_fixed_point_without_forcing():
    """test_d3q19.cpp:131-137."""
    f = np.tile(equilibrium(1.0, (0.01, -0.02, 0.005)), (N ** 3, 1))
    out = device_collide(f, lbm.TrtParams.from_tau(0.9), (0.0, 0.0, 0.0))
    assert np.allclose(out, f, rtol=1e-14, atol=0)


@gpu
def test_trt_collide_conserves_mass_and_momentum_over_random_states():
    """test_d3q19.cpp:139-154."""
    f = random_states(42)
    out = device_collide(f, lbm.TrtParams.from_tau(0.8), (0.0, 0.0, 0.0))
    rho = f.sum(axis=1)
    assert np.all(np.abs((out - f).sum(axis=1)) <= 1e-13 * rho)
    assert np.all(np.abs((out - f) @ C) <= 1e-13)


@gpu
def test_trt_collide_adds_rho_g_of_momentum_per_collision():
    """test_d3q19.cpp:156-172."""
    f = random_states(7)
    g = np.array([1e-6, 0.0, 0.0])
    out = device_collide(f, lbm.TrtParams.from_tau(0.9), g)
    assert np.all(np.abs((out - f) @ C - f.sum(axis=1)[:, None] * g) <= 1e-15)


@gpu
def test_collide_node_matches_a_direct_formula_evaluation(port):
    """test_d3q19.cpp:174-205: an independent transcription of the TRT update,
    term by term, to 1e-13 -- and the oracle's collide_node bit for bit."""
    p = lbm.TrtParams.from_tau(1.1)
    wp, wm = p.omega_plus, p.omega_minus()
    g = np.array([2e-6, -1e-6, 3e-6])
    f = random_states(11)
    out = device_collide(f, p, g)
    for n in range(200):
        rho = f[n].sum()
        u = (f[n] @ C) / rho
        feq = equilibrium(rho, u)
        fplus, fminus = 0.5 * (f[n] + f[n][OPP]), 0.5 * (f[n] - f[n][OPP])
        eplus, eminus = 0.5 * (feq + feq[OPP]), 0.5 * (feq - feq[OPP])
        expect = f[n] - wp * (fplus - eplus) - wm * (fminus - eminus) + 3.0 * W * rho * (C @ g)
        assert np.allclose(out[n], expect, rtol=1e-13, atol=0), n
    for n in range(N ** 3):
        assert np.array_equal(out[n], port.collide(f[n], wp, wm, g)), n

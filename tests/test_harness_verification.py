"""The reference's harness and verification tests (proj/tests/test_harness.cpp,
proj/tests/test_verification.cpp), case by case, against the GPU library:
run_benchmark through the lbmbench-gpu CLI (tools/lbmbench_gpu.cpp), the
steady-state driver and the Poiseuille verification through the C ABI.

Not mirrored: the worker-pool cases (affinity records, LBMBENCH_MAX_WORKERS:
test_harness.cpp:84-110) -- the CPU pool is out of scope;
the GPU analogue of "worker count must not change the fields" is the number
of parts a lattice is cut into.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1711_11468_b200 as lbm

gpu = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1711_11468_b200", "bin", "lbmbench-gpu")
TAU09 = lbm.TrtParams.from_tau(0.9)
NO_FORCE = lbm.BodyForce((0.0, 0.0, 0.0))


def bench(kernel, iterations=10, extra=()):
    """small_config (test_harness.cpp:11-21): blocks 12x10x10, 10 iterations,
    warmup 2, g = (1e-6, 0, 0), seed 31337."""
    return subprocess.run([CLI, "bench", "--kernel", kernel, "--geometry", "blocks", "--dims",
                           "12x10x10", "--block", "4", "--spacing", "4", "--iterations",
                           str(iterations), "--warmup", "2", "--gx", "1e-6", "--seed", "31337",
                           "--format", "json", *extra], capture_output=True, text=True, timeout=600)


# ---- test_harness.cpp --------------------------------------------------------
@gpu
def test_mflups_arithmetic():
    """test_harness.cpp:25-33."""
    r = bench("list-aa-soa")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["n_fluid"] == 1136  # 12*10*10 - 4^3
    assert j["mflups"] == pytest.approx(j["n_fluid"] * j["iterations"] / j["seconds"] / 1e6,
                                        rel=1e-5)
    assert 4802000.0 * 100 / 10.0 / 1e6 == pytest.approx(48.02)


def test_config_validation_happens_before_allocation():
    """test_harness.cpp:35-44: odd iterations with an AA kernel and zero
    iterations are configuration errors (exit 1) -- raised before any device
    work, so this runs without a GPU."""
    for it in (5, 0):
        r = bench("aa-soa", iterations=it)
        assert r.returncode == 1, (it, r.stderr)
        assert "configuration error" in r.stderr


@gpu
def test_rerunning_a_seeded_config_reproduces_the_final_state_bitwise():
    """test_harness.cpp:46-57; "worker count must not change the fields" ->
    2 and 4 node-range parts of the same lattice."""
    a, b = json.loads(bench("list-pull-soa").stdout), json.loads(bench("list-pull-soa").stdout)
    assert a["state_hash"] == b["state_hash"] and a["n_fluid"] == b["n_fluid"] == 1136
    # the same job through the library: seed 31337, warmup 2 + 10 iterations
    spec = lbm.GeometrySpec("blocks", 12, 10, 10, 4, 4)
    force = lbm.BodyForce((1e-6, 0.0, 0.0))
    hashes = []
    for name, dist in (("list-pull-soa", None), ("list-aa-soa", None),
                       ("list-aa-soa", {"virtual_parts": 2}), ("list-aa-soa", {"virtual_parts": 4})):
        k = lbm.make_kernel(lbm.make_descriptor(name), spec, dist=dist)
        k.load_perturbed(31337)
        k.advance(TAU09, force, 12)  # the CLI's default tau
        hashes.append("%016x" % k.fingerprint())
    assert hashes[0] == a["state_hash"]
    assert hashes[1] == hashes[2] == hashes[3]


@gpu
def test_v_fraction_is_reported_for_run_coded_kernels_only():
    """test_harness.cpp:75-82."""
    spec = lbm.GeometrySpec("blocks", 12, 10, 10, 4, 4)
    v = lbm.make_kernel(lbm.make_descriptor("list-aa-pv-soa"), spec).vector_fraction()
    assert v is not None and 0.0 <= v <= 1.0
    assert lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), spec).vector_fraction() is None


@gpu
def test_steady_state_run_returns_after_one_interval_on_a_settled_field():
    """test_harness.cpp:112-123: g = 0 from equilibrium, nothing moves."""
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("slit", 4, 4, 8))
    r = k.steady_state_run(TAU09, NO_FORCE, 10, 1e-12, 1000)
    assert r == {"steps": 10, "converged": True, "final_delta": 0.0}


@gpu
def test_steady_state_run_reports_divergence():
    """test_harness.cpp:125-136."""
    k = lbm.make_kernel(lbm.make_descriptor("blk-push-soa"), lbm.GeometrySpec("slit", 4, 4, 8),
                        lbm.PaddingPolicy.none())
    bad = np.full(k.n_fluid() * 19, 0.05)
    bad[7] = np.nan
    k.load_state(bad)
    with pytest.raises(lbm.NumericalError):
        k.steady_state_run(TAU09, NO_FORCE, 4, 1e-12, 100)


@gpu
def test_steady_state_run_converges_on_the_slit_flow():
    """test_harness.cpp:138-149."""
    k = lbm.make_kernel(lbm.make_descriptor("list-aa-soa"), lbm.GeometrySpec("slit", 4, 4, 18))
    r = k.steady_state_run(TAU09, lbm.BodyForce((1e-6, 0.0, 0.0)), 200, 1e-11, 100000)
    assert r["converged"] and 200 < r["steps"] < 100000


def test_perturbed_equilibrium_is_deterministic_and_physical():
    """test_harness.cpp:151-163 (host function)."""
    a, b, c = (lbm.perturbed_equilibrium(100, s) for s in (7, 7, 8))
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    w = np.tile([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12, 100)
    assert np.all(a > 0.0) and np.all(np.abs(a / w - 1.0) <= 5.1e-4)


@gpu
def test_device_perturbed_init_equals_the_host_function():
    """load_perturbed (the harness's seeded init on the device,
    harness.cpp:50-62) writes exactly perturbed_equilibrium(n_fluid, seed)."""
    for name in ("aa-soa", "list-pull-aos"):
        k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec("pipe", 9, 12, 13))
        k.load_perturbed(31337)
        assert np.array_equal(k.snapshot(), lbm.perturbed_equilibrium(k.n_fluid(), 31337)), name


# ---- test_verification.cpp ---------------------------------------------------
def test_analytic_profile_walls_centerline_symmetry():
    """test_verification.cpp:10-38: 8x8x34, g = 1e-6, tau+ = 0.9 -> nu = 2/15,
    h = 32; the layer maximum sits at zeta = 15.5."""
    c = lbm.PoiseuilleCase()
    u = lbm.analytic_profile(c)
    assert u.size == 32
    assert u.max() == pytest.approx(9.6e-4 * 255.75 / 256.0, rel=1e-12)
    h, nu = 32.0, 2.0 / 15.0
    zeta = np.arange(32) + 0.5
    assert np.allclose(u, c.g / (2 * nu) * zeta * (h - zeta), rtol=1e-14, atol=0)
    assert np.allclose(u, u[::-1], rtol=1e-14, atol=0)
    assert c.g * h * h / (8 * nu) == pytest.approx(9.6e-4, rel=1e-12)
    assert c.params.viscosity() == pytest.approx(nu, rel=1e-15)


def test_case_validation():
    """test_verification.cpp:40-47: nz < 6 and a sonic centerline velocity are
    configuration errors (before any device work)."""
    with pytest.raises(lbm.ConfigError, match="nz must be >= 6"):
        lbm.verify_kernel("list-aa-soa", lbm.PoiseuilleCase(8, 8, 4))
    with pytest.raises(lbm.ConfigError, match="speed of sound"):
        lbm.verify_kernel("list-aa-soa", lbm.PoiseuilleCase(8, 8, 34, 1.0))


@gpu
def test_zero_forcing_gives_a_zero_profile_with_zero_error():
    """test_verification.cpp:49-61."""
    rep = lbm.verify_kernel("list-aa-soa", lbm.PoiseuilleCase(4, 4, 10, 0.0), 10, 1e-13, 1000)
    assert rep["converged"] and rep["passed"]
    assert rep["linf_rel"] == 0.0 and rep["l2_rel"] == 0.0
    assert all(v == 0.0 for v in rep["simulated_ux"])


@gpu
def test_one_kernel_per_family_passes_a_small_slit_case():
    """test_verification.cpp:63-76: h = 16, far below the 1e-4 gate."""
    c = lbm.PoiseuilleCase(4, 4, 18)
    for name in ("list-aa-pv-soa", "blk-pull-soa"):
        rep = lbm.verify_kernel(name, c, 200, 1e-12, 60000)
        assert rep["converged"] and rep["passed"], name
        assert rep["linf_rel"] < 1e-6
        assert rep["half_force_shift"] == c.g / 2


@gpu
def test_simulated_slit_profile_is_x_and_y_invariant():
    """test_verification.cpp:78-100: snapshot order is column-major (x, y),
    z innermost; every column carries the same profile to 1e-13."""
    c = lbm.PoiseuilleCase(5, 6, 14)
    k = lbm.make_kernel(lbm.make_descriptor("list-push-soa"), lbm.GeometrySpec("slit", 5, 6, 14))
    k.steady_state_run(c.params, lbm.BodyForce((c.g, 0.0, 0.0)), 100, 1e-10, 40000)
    _, u = lbm.macro_fields(k.snapshot())
    layers = c.fluid_layers()
    ux = np.asarray(u).reshape(-1, 3)[:, 0].reshape(c.nx * c.ny, layers)
    assert np.all(np.abs(ux - ux[0]) <= 1e-13 * np.maximum(np.abs(ux[0]), 1e-30))


@gpu
def test_verification_agrees_with_the_reference_steppers_target(port):
    """test_verification.cpp:102-132: the textbook half-way stepper (the
    oracle's) establishes the expected profile independently: after 12,000
    steps on the 4x4x14 slit it sits within 1e-4 of the analytic profile, and
    the GPU's steady profile sits on the stepper's."""
    c = lbm.PoiseuilleCase(4, 4, 14)
    snap, _ = port.run("half", "slit", 4, 4, 14, 12000, c.params.omega_plus, g=(c.g, 0.0, 0.0))
    _, u = port.macro(snap)
    layers = c.fluid_layers()
    prof = u[:, 0].reshape(c.nx * c.ny, layers).sum(axis=0) / (c.nx * c.ny) + c.g / 2
    ana = lbm.analytic_profile(c)
    assert np.max(np.abs(prof - ana)) / np.max(np.abs(ana)) < 1e-4
    rep = lbm.verify_kernel("list-aa-soa", c, 200, 1e-12, 60000)
    assert rep["converged"] and rep["passed"]
    assert np.max(np.abs(np.asarray(rep["simulated_ux"]) - prof)) / np.max(np.abs(ana)) < 1e-6

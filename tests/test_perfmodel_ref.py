"""The reference's performance-model tests (proj/tests/test_perfmodel.cpp) for
the parts on the hot path's surface: loop_balance (with and without run
statistics), roofline and micro_for -- host arithmetic through the C ABI, no
device call.  The model report, the bandwidth-set files (:102-148) and the
CPU micro-benchmark protocol are out of scope; the
byte accounting of the device micro-benchmarks is tests/test_microbench.py."""
import pytest

import paper_1711_11468_b200 as lbm


def test_loop_balance_reproduces_every_table_entry():
    """test_perfmodel.cpp:11-32."""
    expect = {"blk-push-aos": 456, "blk-push-soa": 456, "blk-pull-aos": 456, "blk-pull-soa": 456,
              "aa-aos": 304, "aa-soa": 304, "aa-vec-soa": 304, "list-push-aos": 528,
              "list-push-soa": 528, "list-pull-aos": 528, "list-pull-soa": 528,
              "list-pull-split-nt-1s-soa": 376, "list-pull-split-nt-2s-soa": 376,
              "list-aa-aos": 340, "list-aa-soa": 340}
    for name, value in expect.items():
        lo, hi, _ = lbm.loop_balance(name)
        assert lo == hi == value, name  # not a range
    for name in ("list-aa-ria-soa", "list-aa-pv-soa"):
        lo, hi, _ = lbm.loop_balance(name)
        assert (lo, hi) == (304, 342), name  # a range without run statistics


def test_ria_loop_balance_hits_both_endpoints_and_the_channel_point():
    """test_perfmodel.cpp:34-46."""
    ria = "list-aa-ria-soa"
    assert lbm.loop_balance(ria, {"total_runs": 0, "n_fluid": 1000})[0] == pytest.approx(304.0, rel=1e-12)
    assert lbm.loop_balance(ria, {"total_runs": 1000, "n_fluid": 1000})[0] == pytest.approx(342.0, rel=1e-12)
    lo, hi, _ = lbm.loop_balance(ria, {"total_runs": 3, "n_fluid": 98})
    assert lo == hi and abs(lo - 305.2) < 0.05
    # the statistics only matter for the run-coded names
    assert lbm.loop_balance("list-aa-soa", {"total_runs": 3, "n_fluid": 98}) == lbm.loop_balance("list-aa-soa")


def test_loop_balance_breakdown_adds_up():
    """test_perfmodel.cpp:48-56: B_l = 152 read + 152 written + write allocate
    (one-step kernels without streaming stores) + index bytes."""
    for name in lbm.kernel_names():
        d = lbm.make_descriptor(name)
        lo, hi, gpu = lbm.loop_balance(name)
        os_ = d.prop != "aa"
        wa = 152 if os_ and d.nt_streams == 0 else 0
        if d.addr == "direct":
            index = (0, 0)
        elif d.ria:
            index = (0, 38)
        else:
            index = (72, 72) if os_ else (36, 36)
        assert (lo, hi) == (304 + wa + index[0], 304 + wa + index[1]), name
        # the GPU never pays the write allocate
        assert gpu == 304 + (0.5 if d.ria else index[0]), name


def test_roofline_arithmetic():
    """test_perfmodel.cpp:58-72."""
    lo, hi, _ = lbm.loop_balance("list-pull-aos")
    assert lbm.roofline(48.0, lo, hi)[0] == pytest.approx(90.909, rel=1e-3)
    lo, hi, _ = lbm.loop_balance("aa-soa")
    assert lbm.roofline(51.1, lo, hi)[0] == pytest.approx(168.1, rel=1e-3)
    for bad in (0.0, -1.0):
        with pytest.raises(lbm.ConfigError):
            lbm.roofline(bad, lo, hi)


def test_roofline_is_monotone_in_b_and_bl():
    """test_perfmodel.cpp:74-88."""
    lo = lbm.loop_balance("aa-soa")[:2]          # 304
    hi = lbm.loop_balance("list-pull-soa")[:2]   # 528
    assert lbm.roofline(50.0, *lo)[0] > lbm.roofline(40.0, *lo)[0]
    assert lbm.roofline(50.0, *lo)[0] > lbm.roofline(50.0, *hi)[0]
    pmin, pmax = lbm.roofline(50.0, *lbm.loop_balance("list-aa-ria-soa")[:2])
    assert pmin < pmax  # range in, range out
    assert pmin == pytest.approx(50.0 * 1000 / 342) and pmax == pytest.approx(50.0 * 1000 / 304)


def test_kernel_to_micro_benchmark_mapping_follows_the_table():
    """test_perfmodel.cpp:90-100."""
    expect = {"blk-push-aos": "copy-19", "list-pull-soa": "copy-19",
              "list-pull-split-nt-1s-soa": "copy-19-nt-sl",
              "list-pull-split-nt-2s-soa": "copy-19-nt-sl", "aa-aos": "update-19",
              "aa-vec-soa": "update-19", "list-aa-pv-soa": "update-19"}
    for name, kind in expect.items():
        assert lbm.micro_for(lbm.make_descriptor(name)) == kind, name

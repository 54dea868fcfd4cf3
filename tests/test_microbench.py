"""Device micro-benchmarks: byte accounting against the
reference's run_microbench (microbench.cpp:92-99) and, on the GPU, the
measured ceilings used for roofline.adjusted in bench.py."""
import json
import os

import pytest

import paper_1711_11468_b200 as lbm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = ["copy", "copy-19", "copy-19-nt-sl", "update-19"]


@pytest.mark.parametrize("kind", KINDS)
def test_accounting_matches_reference(kind):
    """One pass over the same working set: the reference's accounted bytes
    (its own run_microbench, oracle/_ref) equal lbmgpu's `bytes_ref`, and the
    GPU accounting drops exactly the 8 B write allocate per element and
    stream for the plain copies (GPU full-sector stores allocate nothing)."""
    try:
        from oracle.oracle import Ref
        ref = Ref()
    except FileNotFoundError:
        pytest.skip("reference library not built")
    ws = 4 * ref.llc_bytes()
    ws += (-ws) % (38 * 16)  # whole double2 per stream for every kind
    acc = lbm.lbmgpu.microbench_accounting(kind, ws)
    ref_bytes, passes, _ = ref.microbench(kind, ws)
    assert passes >= 1
    assert acc["bytes_ref"] == ref_bytes
    streams = 1 if kind == "copy" else 19
    wa = 8 * streams * acc["elems"] if kind in ("copy", "copy-19") else 0
    assert acc["bytes_gpu"] == ref_bytes - wa
    assert acc["bytes_gpu"] == 16 * streams * acc["elems"]


def test_accounting_rejects_unknown_kind():
    with pytest.raises(lbm.ConfigError, match="valid: copy"):
        lbm.lbmgpu.microbench_accounting("triad", 1 << 30)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["copy-19", "update-19"])
def test_device_microbench_ceiling(kind):
    """The measured ceiling is a plausible fraction of the pool's measured
    copy peak (MEASURED_PEAKS.json; 6.55 TB/s fallback): the 19-stream
    kernels reach 0.8-1.15 of it at a 32 GiB working set."""
    peak = 6549.8
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = float(json.load(open(p))["hbm_gbs"])
    gbps = lbm.lbmgpu.microbench(kind, 32 << 30, 3)
    assert 0.8 * peak <= gbps <= 1.15 * peak, (kind, gbps, peak)

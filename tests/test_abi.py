"""CPU: the C-ABI library loads, exports every symbol include/lbmgpu.h
declares, and its host-only logic (registry, padding, loop balance, halo plan,
fingerprint) behaves like the reference.  No compute call here needs a GPU;
compute calls without a device must fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1711_11468_b200 as lbm
from paper_1711_11468_b200 import lbmgpu as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lbmgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lbmgpu_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 30
    so = ctypes.CDLL(L.LIB_PATH)
    missing = [s for s in syms if not hasattr(so, s)]
    assert not missing, missing
    assert so.lbmgpu_abi_version() == 2


def test_kernel_names_order():
    assert lbm.kernel_names() == [
        "blk-push-aos", "blk-push-soa", "blk-pull-aos", "blk-pull-soa", "aa-aos", "aa-soa",
        "aa-vec-soa", "list-push-aos", "list-push-soa", "list-pull-aos", "list-pull-soa",
        "list-pull-split-nt-1s-soa", "list-pull-split-nt-2s-soa", "list-aa-aos", "list-aa-soa",
        "list-aa-ria-soa", "list-aa-pv-soa"]


def test_descriptors_like_reference():
    """tests/test_kernels.cpp:29-54."""
    nt = lbm.make_descriptor("list-pull-split-nt-2s-soa")
    assert (nt.prop, nt.addr, nt.layout, nt.nt_streams) == ("os-pull", "indirect", "soa", 2)
    pv = lbm.make_descriptor("list-aa-pv-soa")
    assert pv.prop == "aa" and pv.ria and pv.pv
    vec = lbm.make_descriptor("aa-vec-soa")
    assert vec.vec and vec.addr == "direct"
    with pytest.raises(lbm.ConfigError) as e:
        lbm.make_descriptor("plain-push")
    assert "blk-push-aos" in str(e.value) and "list-aa-pv-soa" in str(e.value)
    with pytest.raises(lbm.ConfigError):
        lbm.make_descriptor("aa-soa", blk=-1)
    with pytest.raises(lbm.ConfigError):
        lbm.make_descriptor("aa-soa", vector_width=9)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblbm_ref.so")),
                    reason="reference library not built here")
def test_descriptors_equal_reference_library():
    from oracle.oracle import Ref
    ref = Ref()
    for name in ref.kernel_names():
        r = ref.descriptor(name, 3)
        d = lbm.make_descriptor(name, 3)
        assert ["os-push", "os-pull", "aa"][r["prop"]] == d.prop
        assert bool(r["layout_soa"]) == (d.layout == "soa")
        assert bool(r["indirect"]) == (d.addr == "indirect")
        assert (r["nt"], bool(r["ria"]), bool(r["pv"]), bool(r["vec"])) == \
            (d.nt_streams, d.ria, d.pv, d.vec)
        assert ref.loop_balance(name)[0] == lbm.loop_balance(name)[0] or d.ria


def test_loop_balance_table1():
    """Reference B_l (tests/test_perfmodel.cpp:11-32) and the
    GPU algorithmic bytes (no write allocate)."""
    exp = {"blk-push-soa": (456, 304), "aa-soa": (304, 304), "list-pull-soa": (528, 376),
           "list-pull-split-nt-1s-soa": (376, 376), "list-aa-soa": (340, 340),
           "list-push-aos": (528, 376)}
    for name, (ref_bl, gpu) in exp.items():
        a, b, g = lbm.loop_balance(name)
        assert a == b == ref_bl and g == gpu, name
    a, b, g = lbm.loop_balance("list-aa-ria-soa")
    assert (a, b, g) == (304, 342, 304.5)  # GPU: one-byte pattern id per odd sub-step


def test_padding_against_golden(small_golden):
    for p in small_golden["padding"]:
        st, tot = lbm.padding_offsets(p["n_fluid"], lbm.PaddingPolicy(p["mode"]))
        assert [int(v) for v in st] == p["starts"] and tot == p["total"]
    st, tot = lbm.padding_offsets(10, lbm.PaddingPolicy.parse(",".join(["3"] * 19)))
    assert int(st[0]) == 3 and int(st[1]) == 16 and tot == 19 * 13
    with pytest.raises(lbm.ConfigError):
        lbm.PaddingPolicy.parse("1,2,3")
    with pytest.raises(lbm.ConfigError):
        lbm.PaddingPolicy.parse("x" + ",0" * 18)


def test_fingerprint_known_answer(port):
    a = np.linspace(0, 1, 999)
    assert lbm.state_fingerprint(a) == port.fingerprint(a)
    assert lbm.state_fingerprint(np.zeros(0)) == 0xcbf29ce484222325


def test_omega_minus():
    """d3q19.hpp:70-73: tau=1, Lambda=3/16 -> omega- = 8/7."""
    assert abs(lbm.TrtParams(1.0).omega_minus() - 8.0 / 7.0) < 1e-15


def test_halo_plan_invariants():
    for nz, parts, ring in [(512, 8, False), (16, 4, True), (17, 5, False), (4, 2, True)]:
        rows = L.halo_plan(nz, parts, ring)
        nb = parts if ring else parts - 1
        assert rows.shape == (4 * nb, 7)
        nzl = [nz * (p + 1) // parts - nz * p // parts for p in range(parts)]
        for ph, src, dst, sp, dp, slot0, nslots in rows:
            assert nslots == 5 and slot0 in (0, 14) and src != dst
            if ph == 0:
                # own boundary plane -> neighbour's ghost plane
                assert 1 <= sp <= nzl[src] and dp in (0, nzl[dst] + 1)
            else:
                assert sp in (0, nzl[src] + 1) and 1 <= dp <= nzl[dst]
            # up slots travel to the top ghost / come from the top ghost
            if slot0 == 14:
                assert (ph == 0 and dp == nzl[dst] + 1) or (ph == 1 and sp == nzl[src] + 1)
            else:
                assert (ph == 0 and dp == 0) or (ph == 1 and sp == 0)


def test_one_step_halo_plan_invariants():
    """Push/pull z-slab plan (halo.hpp phases 2/3): every boundary incl. the
    z ring; pull copies own boundary planes into the neighbour's ghost
    planes (the slots its boundary nodes gather across the face), push
    ships both 5-slot groups of a ghost plane into the neighbour's staging
    plane (-1 bottom / -2 top)."""
    for nz, parts in [(24, 2), (17, 5), (13, 13), (64, 8)]:
        rows = L.halo_plan(nz, parts, True, one_step=True)
        assert rows.shape == (6 * parts, 7)
        nzl = [nz * (p + 1) // parts - nz * p // parts for p in range(parts)]
        pull = rows[rows[:, 0] == 2]
        push = rows[rows[:, 0] == 3]
        assert len(pull) == 2 * parts and len(push) == 4 * parts
        for _, src, dst, sp, dp, slot0, n in pull:
            assert n == 5 and src != dst or parts == 1
            if dp == 0:  # below -> my bottom ghost: the c_z=+1 slots of its top plane
                assert slot0 == 14 and sp == nzl[src] and (dst - src) % parts == 1
            else:        # above -> my top ghost: the c_z=-1 slots of its plane 1
                assert dp == nzl[dst] + 1 and slot0 == 0 and sp == 1 and (src - dst) % parts == 1
        recv = {}
        for _, src, dst, sp, dp, slot0, n in push:
            assert dp in (-1, -2) and slot0 in (0, 14)
            if dp == -1:
                assert sp == nzl[src] + 1 and (dst - src) % parts == 1
            else:
                assert sp == 0 and (src - dst) % parts == 1
            recv.setdefault((int(dst), int(dp)), set()).add(int(slot0))
        # each part's two staging planes receive both slot groups once
        assert recv == {(p, f): {0, 14} for p in range(parts) for f in (-1, -2)}


def test_compute_without_gpu_fails_loudly():
    """No CPU fallback: on a machine without a CUDA device every compute entry
    point raises DeviceError."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(lbm.DeviceError):
        lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", 8, 6, 6))
    with pytest.raises(lbm.DeviceError):
        lbm.build_geometry(lbm.GeometrySpec("channel", 8, 6, 6))


def test_run_entry_validates_without_device():
    """lbmgpu_run (the pipelined job) rejects a missing context with the
    ConfigError status before touching a device."""
    g = (ctypes.c_double * 3)(1e-5, 0.0, 0.0)
    piped = ctypes.c_int(7)
    rc = L.lib.lbmgpu_run(None, 1.0, 3.0 / 16.0, g, 2, None, 0, None, 0, ctypes.byref(piped))
    assert rc == 1
    assert "ctx" in L.lib.lbmgpu_last_error().decode()


def test_config_errors_before_device_work():
    """ConfigError is raised before any device allocation (harness.cpp:84-93):
    these fail with ConfigError even without a GPU."""
    d = lbm.make_descriptor("aa-soa")
    for spec in [lbm.GeometrySpec("channel", 8, 2, 6), lbm.GeometrySpec("blocks", 8, 8, 8, 6, 4),
                 lbm.GeometrySpec("pipe", 8, 3, 8), lbm.GeometrySpec("blocks", 8, 8, 8, 0, 4)]:
        with pytest.raises(lbm.ConfigError):
            lbm.make_kernel(d, spec)
    with pytest.raises(lbm.ConfigError):
        lbm.make_kernel(d, lbm.GeometrySpec("channel", 8, 8, 8), row_pad=-1)
    for name, blk in (("list-pull-soa", 0), ("list-aa-ria-soa", 0), ("list-aa-soa", 2)):
        with pytest.raises(lbm.ConfigError):
            lbm.make_kernel(lbm.make_descriptor(name, blk=blk),
                            lbm.GeometrySpec("channel", 8, 8, 8), dist={"virtual_parts": 2})

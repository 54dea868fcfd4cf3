"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU oracles.

* ``Port``: our C restatement (oracle/lbm_oracle.c -> liblbm_oracle.so).
* ``Ref``:  the unmodified reference lbmbench library compiled from
  /root/reference/proj/src (oracle/_ref/liblbm_ref.so, via oracle/ref_driver.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liblbm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblbm_ref.so")

KINDS = {"channel": 0, "slit": 1, "pipe": 2, "blocks": 3}
PADDING = {"none": 0, "auto": 1, "thrash": 2, "explicit": 3}
Q = 19

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def _pads_arr(pads):
    if pads is None:
        return np.zeros(Q, np.int64)
    return np.ascontiguousarray(pads, dtype=np.int64)


class Port:
    """Our C restatement of the reference algorithm (see lbm_oracle.h)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.ora_collide_node.argtypes = [_dp, C.c_double, C.c_double, _dp]
        L.ora_omega_minus.restype = C.c_double
        L.ora_omega_minus.argtypes = [C.c_double, C.c_double]
        L.ora_geometry.argtypes = [C.c_int] * 7 + [_u8, C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        L.ora_padding_offsets.argtypes = [C.c_uint64, C.c_int, _i64, _u64, C.POINTER(C.c_uint64)]
        L.ora_order_nodes.restype = C.c_int64
        L.ora_order_nodes.argtypes = [_u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ora_build_adjacency.argtypes = [_u8, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                                          _i32, _u32, C.c_int64, C.c_int, _u64, C.c_int, _u32]
        L.ora_perturbed.argtypes = [C.c_uint64, C.c_uint64, C.c_double, _dp]
        L.ora_fingerprint.restype = C.c_uint64
        L.ora_fingerprint.argtypes = [_dp, C.c_uint64]
        L.ora_fingerprint_u32.restype = C.c_uint64
        L.ora_fingerprint_u32.argtypes = [_u32, C.c_uint64]
        L.ora_run.argtypes = [C.c_int, _u8, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                              C.c_void_p, C.c_long, C.c_double, C.c_double, _dp, _dp,
                              C.POINTER(C.c_double)]
        L.ora_macro.argtypes = [_dp, C.c_uint64, _dp, _dp]
        L.ora_max_rel_diff.restype = C.c_double
        L.ora_max_rel_diff.argtypes = [_dp, _dp, C.c_uint64]
        self.L = L

    # -- model
    def collide(self, f, wp, wm, g):
        f = np.array(f, dtype=np.float64)
        self.L.ora_collide_node(f, wp, wm, np.asarray(g, np.float64))
        return f

    def omega_minus(self, wp, lam=3.0 / 16.0):
        return self.L.ora_omega_minus(wp, lam)

    # -- geometry
    def geometry(self, kind, nx, ny, nz, block=4, spacing=4, pipe_diameter=0):
        flags = np.zeros(nx * ny * nz, np.uint8)
        per = (C.c_int * 3)()
        nf = C.c_int64(0)
        rc = self.L.ora_geometry(KINDS[kind], nx, ny, nz, block, spacing, pipe_diameter,
                                 flags, per, C.byref(nf))
        if rc:
            raise ValueError(f"geometry {kind} {nx}x{ny}x{nz}: config error")
        return flags, tuple(per), int(nf.value)

    def padding_offsets(self, n_fluid, mode="auto", pads=None):
        starts = np.zeros(Q, np.uint64)
        tot = C.c_uint64(0)
        self.L.ora_padding_offsets(n_fluid, PADDING[mode], _pads_arr(pads), starts, C.byref(tot))
        return starts, int(tot.value)

    def structure(self, kind, nx, ny, nz, block=4, spacing=4, pipe_diameter=0,
                  layout="soa", blk=0, padding="auto", pads=None, scatter=False):
        flags, per, nf = self.geometry(kind, nx, ny, nz, block, spacing, pipe_diameter)
        nodes = np.zeros(3 * nf, np.int32)
        rank = np.zeros(nx * ny * nz, np.uint32)
        n = self.L.ora_order_nodes(flags, nx, ny, nz, blk, nodes.ctypes.data, rank.ctypes.data)
        assert n == nf
        if layout == "soa":
            starts, total = self.padding_offsets(nf, padding, pads)
        else:
            starts, total = np.zeros(Q, np.uint64), nf * Q
        adj = np.zeros(nf * 18, np.uint32)
        perc = (C.c_int * 3)(*per)
        self.L.ora_build_adjacency(flags, perc, nx, ny, nz, nodes, rank, nf,
                                   1 if layout == "soa" else 0, starts, 1 if scatter else 0, adj)
        return dict(n_fluid=nf, nodes=nodes.reshape(-1, 3), rank=rank, starts=starts,
                    total_slots=total, adj=adj)

    # -- state helpers
    def perturbed(self, n_fluid, seed, amplitude=1e-3):
        out = np.zeros(n_fluid * Q, np.float64)
        self.L.ora_perturbed(n_fluid, seed, amplitude, out)
        return out

    def fingerprint(self, a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint32:
            return int(self.L.ora_fingerprint_u32(a, a.size))
        return int(self.L.ora_fingerprint(np.ascontiguousarray(a, np.float64), a.size))

    def run(self, family, kind, nx, ny, nz, steps, omega_plus, magic_lambda=3.0 / 16.0,
            g=(0.0, 0.0, 0.0), init=None, block=4, spacing=4, pipe_diameter=0):
        """family 'full' (full-way bounce-back, direct kernels) or 'half'
        (half-way, list kernels).  Returns (canonical snapshot, mass)."""
        flags, per, nf = self.geometry(kind, nx, ny, nz, block, spacing, pipe_diameter)
        out = np.zeros(nf * Q, np.float64)
        mass = C.c_double(0.0)
        wm = self.omega_minus(omega_plus, magic_lambda)
        initp = None
        if init is not None:
            init = np.ascontiguousarray(init, np.float64)
            assert init.size == nf * Q
            initp = init.ctypes.data
        perc = (C.c_int * 3)(*per)
        rc = self.L.ora_run(0 if family == "full" else 1, flags, perc, nx, ny, nz, initp, steps,
                            omega_plus, wm, np.asarray(g, np.float64), out, C.byref(mass))
        if rc:
            raise MemoryError("oracle run failed")
        return out, mass.value

    def macro(self, snap):
        n = snap.size // Q
        rho = np.zeros(n)
        u = np.zeros(3 * n)
        self.L.ora_macro(np.ascontiguousarray(snap, np.float64), n, rho, u)
        return rho, u.reshape(-1, 3)

    def max_rel_diff(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        assert a.size == b.size
        return self.L.ora_max_rel_diff(a, b, a.size)


def _fnv_bytes(b: np.ndarray) -> int:
    """FNV-1a 64 over a uint8 array, via the port library's C loop."""
    P = Port()
    return int(P.L.ora_fingerprint_u32(np.ascontiguousarray(b).view(np.uint32), b.size // 4)) \
        if b.size % 4 == 0 else _fnv_py(b)


def _fnv_py(b):
    h = 0xcbf29ce484222325
    for x in b.tobytes():
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Ref:
    """The unmodified reference (oracle/_ref/liblbm_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_geometry.argtypes = [C.c_int] * 7 + [C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.ref_create.argtypes = [C.c_char_p] + [C.c_int] * 9 + [C.c_void_p, C.c_int, C.c_int,
                                                                 C.c_void_p, C.c_int,
                                                                 C.POINTER(C.c_void_p)]
        L.ref_pinned.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.ref_microbench.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_llc_bytes.restype = C.c_uint64
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_n_fluid.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.ref_load_state.argtypes = [C.c_void_p, _dp, C.c_uint64]
        L.ref_snapshot.argtypes = [C.c_void_p, _dp, C.c_uint64]
        L.ref_fingerprint_state.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.ref_total_mass.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.ref_advance.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, C.c_long,
                                  C.POINTER(C.c_double)]
        L.ref_ria_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_structure.argtypes = ([C.c_int] * 10 +[C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]
                                    + [C.c_void_p] * 3 + [C.POINTER(C.c_uint64)])
        L.ref_ria.argtypes = [C.c_int] * 8 + [C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_padding_offsets.argtypes = [C.c_uint64, C.c_int, _i64, _u64, C.POINTER(C.c_uint64)]
        L.ref_perturbed.argtypes = [C.c_uint64, C.c_uint64, C.c_double, _dp]
        L.ref_fingerprint.restype = C.c_uint64
        L.ref_fingerprint.argtypes = [_dp, C.c_uint64]
        L.ref_collide_node.argtypes = [_dp, C.c_double, C.c_double, _dp]
        L.ref_descriptor.argtypes = [C.c_char_p, C.c_int] + [C.POINTER(C.c_int)] * 7
        L.ref_loop_balance.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_kernel_names.argtypes = [C.c_char_p, C.c_uint64]
        L.ref_verify.argtypes = ([C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                  C.c_double, C.c_int, C.c_long, C.c_double, C.c_long]
                                 + [C.POINTER(C.c_double)] * 2 + [C.POINTER(C.c_long)]
                                 + [C.POINTER(C.c_int)] * 2 + [C.c_void_p] * 2)
        self.L = L

    def _chk(self, rc):
        if rc:
            raise RefError(rc, self.L.ref_last_error().decode())

    def microbench(self, kind, working_set, workers=2):
        """(bytes accounted per pass, passes, GB/s) of one short repetition
        of the reference's run_microbench."""
        b, p, g = C.c_uint64(), C.c_int(), C.c_double()
        self._chk(self.L.ref_microbench(kind.encode(), working_set, workers, C.byref(b),
                                        C.byref(p), C.byref(g)))
        return b.value, p.value, g.value

    def llc_bytes(self):
        return int(self.L.ref_llc_bytes())

    def kernel_names(self):
        buf = C.create_string_buffer(4096)
        self._chk(self.L.ref_kernel_names(buf, 4096))
        return buf.value.decode().split()

    def descriptor(self, name, blk=0):
        v = [C.c_int() for _ in range(7)]
        self._chk(self.L.ref_descriptor(name.encode(), blk, *[C.byref(x) for x in v]))
        keys = ["prop", "layout_soa", "indirect", "nt", "ria", "pv", "vec"]
        return {k: x.value for k, x in zip(keys, v)}

    def loop_balance(self, name):
        a, b = C.c_double(), C.c_double()
        self._chk(self.L.ref_loop_balance(name.encode(), C.byref(a), C.byref(b)))
        return a.value, b.value

    def geometry(self, kind, nx, ny, nz, block=4, spacing=4, pipe_diameter=0):
        flags = np.zeros(nx * ny * nz, np.uint8)
        nf = C.c_int64()
        per = (C.c_int * 3)()
        self._chk(self.L.ref_geometry(KINDS[kind], nx, ny, nz, block, spacing, pipe_diameter,
                                      flags.ctypes.data, C.byref(nf), C.cast(per, C.c_void_p)))
        return flags, tuple(per), nf.value

    def structure(self, kind, nx, ny, nz, block=4, spacing=4, pipe_diameter=0, layout="soa",
                  blk=0, padding="auto", pads=None, scatter=False):
        nf = C.c_uint64()
        args = (KINDS[kind], nx, ny, nz, block, spacing, pipe_diameter,
                1 if layout == "soa" else 0, blk, PADDING[padding])
        self._chk(self.L.ref_structure(*args, _pads_arr(pads).ctypes.data, int(scatter), C.byref(nf),
                                       None, None, None, None))
        n = nf.value
        nodes = np.zeros(3 * n, np.int32)
        adj = np.zeros(18 * n, np.uint32)
        starts = np.zeros(Q, np.uint64)
        tot = C.c_uint64()
        self._chk(self.L.ref_structure(*args, _pads_arr(pads).ctypes.data, int(scatter), C.byref(nf),
                                       nodes.ctypes.data, adj.ctypes.data, starts.ctypes.data,
                                       C.byref(tot)))
        return dict(n_fluid=n, nodes=nodes.reshape(-1, 3), adj=adj, starts=starts,
                    total_slots=tot.value)

    def ria(self, kind, nx, ny, nz, block=4, spacing=4, blk=0, vector_width=4):
        runs, v = C.c_uint64(), C.c_double()
        self._chk(self.L.ref_ria(KINDS[kind], nx, ny, nz, block, spacing, blk, vector_width,
                                 C.byref(runs), C.byref(v)))
        return runs.value, v.value

    def padding_offsets(self, n_fluid, mode="auto", pads=None):
        starts = np.zeros(Q, np.uint64)
        tot = C.c_uint64()
        self._chk(self.L.ref_padding_offsets(n_fluid, PADDING[mode], _pads_arr(pads), starts,
                                             C.byref(tot)))
        return starts, tot.value

    def perturbed(self, n_fluid, seed, amplitude=1e-3):
        out = np.zeros(n_fluid * Q)
        self._chk(self.L.ref_perturbed(n_fluid, seed, amplitude, out))
        return out

    def fingerprint(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return int(self.L.ref_fingerprint(a, a.size))

    @staticmethod
    def fingerprint_u32(a):
        """FNV-1a over little-endian uint32 bytes (same function as
        harness.cpp:27-39 applied to the adjacency array)."""
        b = np.ascontiguousarray(a, dtype="<u4").view(np.uint8)
        return _fnv_bytes(b)

    def collide(self, f, wp, wm, g):
        f = np.array(f, dtype=np.float64)
        self.L.ref_collide_node(f, wp, wm, np.asarray(g, np.float64))
        return f

    def kernel(self, name, kind, nx, ny, nz, block=4, spacing=4, pipe_diameter=0, blk=0,
               padding="auto", pads=None, threads=1, vector_width=4, pin=None):
        """pin: core ids for the workers (reference --pin, workers.cpp:26-39)."""
        return RefKernel(self, name, kind, nx, ny, nz, block, spacing, pipe_diameter, blk,
                         padding, pads, threads, vector_width, pin)

    def verify(self, name, nx=8, ny=8, nz=34, g=1e-6, tau=0.9, magic_lambda=3.0 / 16.0,
               threads=1, interval=200, tol=1e-12, max_steps=200000):
        linf, l2 = C.c_double(), C.c_double()
        steps = C.c_long()
        conv, passed = C.c_int(), C.c_int()
        sim = np.zeros(nz - 2)
        ana = np.zeros(nz - 2)
        self._chk(self.L.ref_verify(name.encode(), nx, ny, nz, g, tau, magic_lambda, threads,
                                    interval, tol, max_steps, C.byref(linf), C.byref(l2),
                                    C.byref(steps), C.byref(conv), C.byref(passed),
                                    sim.ctypes.data, ana.ctypes.data))
        return dict(linf_rel=linf.value, l2_rel=l2.value, steps=steps.value,
                    converged=bool(conv.value), passed=bool(passed.value), simulated=sim,
                    analytic=ana)


class RefKernel:
    def __init__(self, ref, name, kind, nx, ny, nz, block, spacing, pipe_diameter, blk, padding,
                 pads, threads, vector_width, pin=None):
        self.ref = ref
        self.h = C.c_void_p()
        pin_arr = np.asarray(list(pin or []), np.int32)
        ref._chk(ref.L.ref_create(name.encode(), KINDS[kind], nx, ny, nz, block, spacing,
                                  pipe_diameter, blk, PADDING[padding],
                                  _pads_arr(pads).ctypes.data, threads, vector_width,
                                  pin_arr.ctypes.data if pin_arr.size else None,
                                  int(pin_arr.size), C.byref(self.h)))
        n = C.c_uint64()
        ref._chk(ref.L.ref_n_fluid(self.h, C.byref(n)))
        self.n_fluid = n.value

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.ref.L.ref_destroy(self.h)
            self.h = C.c_void_p()

    def load_state(self, s):
        s = np.ascontiguousarray(s, np.float64)
        self.ref._chk(self.ref.L.ref_load_state(self.h, s, s.size))

    def snapshot(self):
        out = np.zeros(self.n_fluid * Q)
        self.ref._chk(self.ref.L.ref_snapshot(self.h, out, out.size))
        return out

    def fingerprint(self):
        v = C.c_uint64()
        self.ref._chk(self.ref.L.ref_fingerprint_state(self.h, C.byref(v)))
        return v.value

    def total_mass(self):
        v = C.c_double()
        self.ref._chk(self.ref.L.ref_total_mass(self.h, C.byref(v)))
        return v.value

    def pinned(self):
        n = C.c_int()
        self.ref._chk(self.ref.L.ref_pinned(self.h, C.byref(n)))
        return n.value

    def advance(self, omega_plus, magic_lambda, g, steps):
        sec = C.c_double()
        self.ref._chk(self.ref.L.ref_advance(self.h, omega_plus, magic_lambda,
                                             np.asarray(g, np.float64), steps, C.byref(sec)))
        return sec.value

    def ria_stats(self):
        runs, v = C.c_uint64(), C.c_double()
        self.ref._chk(self.ref.L.ref_ria_stats(self.h, C.byref(runs), C.byref(v)))
        return runs.value, (None if v.value < 0 else v.value)

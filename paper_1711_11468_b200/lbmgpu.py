"""Python host mirror of the reference lbmbench kernel/geometry surface,
calling the B200 sweep library (liblbmgpu.so) through its C ABI
(include/lbmgpu.h).

Names, argument meaning and error behaviour follow the reference
(paths relative to /root/reference/proj):

* ``kernel_names`` / ``make_descriptor`` / ``make_kernel``  -- src/kernels.cpp:22-109
* ``Kernel.advance/snapshot/load_state/total_mass/...``      -- include/lbm/kernels.hpp:58-96
* ``TrtParams`` / ``BodyForce``                              -- include/lbm/d3q19.hpp:64-92
* ``GeometrySpec`` / ``build_geometry`` / ``fluid_count``    -- src/geometry.cpp:40-117
* ``PaddingPolicy`` / ``padding_offsets``                    -- src/list_lattice.cpp:10-121
* ``state_fingerprint`` / ``perturbed_equilibrium``         -- src/harness.cpp:27-62
* ``steady_state_run`` / ``verify_kernel``                   -- src/harness.cpp:141-174,
                                                                src/verification.cpp:31-100
* ``ConfigError`` / ``NumericalError``                       -- include/lbm/errors.hpp

There is no CPU fallback: importing this module fails loudly when the CUDA
library has not been built, and every compute call runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

Q = 19
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBMGPU_LIB", os.path.join(_HERE, "liblbmgpu.so"))


class LbmError(RuntimeError):
    pass


class ConfigError(LbmError):
    """lbm::ConfigError (errors.hpp:9-12); CLI exit code 1."""


class NumericalError(LbmError):
    """lbm::NumericalError (errors.hpp:14-17); CLI exit code 2."""


class DeviceError(LbmError):
    """CUDA / NCCL failure (status 4); no reference equivalent."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1711_11468_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, i, u64, i64, d = C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_double
    P = C.POINTER
    L.lbmgpu_last_error.restype = C.c_char_p
    L.lbmgpu_omega_minus.restype = d
    L.lbmgpu_omega_minus.argtypes = [d, d]
    L.lbmgpu_fnv1a.restype = u64
    L.lbmgpu_fnv1a.argtypes = [vp, u64]
    L.lbmgpu_kernel_names.argtypes = [C.c_char_p, C.c_size_t]
    L.lbmgpu_make_descriptor.argtypes = [C.c_char_p, i, i, vp]
    L.lbmgpu_padding_offsets.argtypes = [u64, vp, vp, P(u64)]
    L.lbmgpu_loop_balance.argtypes = [C.c_char_p, P(d), P(d), P(d)]
    L.lbmgpu_loop_balance_stats.argtypes = [C.c_char_p, i64, i64, P(d), P(d), P(d)]
    L.lbmgpu_roofline.argtypes = [d, d, d, P(d), P(d)]
    L.lbmgpu_vectorizable_fraction.argtypes = [vp, i, P(d)]
    L.lbmgpu_export_runs.argtypes = [vp, vp, u64, P(i64)]
    L.lbmgpu_geometry_build.argtypes = [vp, vp, P(i64), vp]
    L.lbmgpu_create.argtypes = [C.c_char_p, i, i, vp, vp, i, vp, P(vp)]
    L.lbmgpu_destroy.argtypes = [vp]
    L.lbmgpu_advance.argtypes = [vp, d, d, vp, C.c_long]
    L.lbmgpu_time_advance.argtypes = [vp, d, d, vp, C.c_long, P(d)]
    L.lbmgpu_n_fluid.argtypes = [vp, P(u64)]
    L.lbmgpu_snapshot.argtypes = [vp, vp, u64]
    L.lbmgpu_load_state.argtypes = [vp, vp, u64]
    L.lbmgpu_run.argtypes = [vp, d, d, vp, C.c_long, vp, u64, vp, u64, P(i)]
    L.lbmgpu_load_perturbed.argtypes = [vp, u64, d]
    L.lbmgpu_total_mass.argtypes = [vp, P(d)]
    L.lbmgpu_fingerprint.argtypes = [vp, P(u64)]
    L.lbmgpu_capabilities.argtypes = [vp, P(i), P(i), P(i)]
    L.lbmgpu_ria_stats.argtypes = [vp, P(i64), P(i64), P(d), P(d)]
    L.lbmgpu_descriptor_of.argtypes = [vp, vp]
    L.lbmgpu_export_structure.argtypes = [vp, vp, vp, vp, P(u64)]
    L.lbmgpu_steady_state_run.argtypes = [vp, d, d, vp, C.c_long, d, C.c_long,
                                          P(C.c_long), P(i), P(d)]
    L.lbmgpu_layer_ux.argtypes = [vp, vp]
    L.lbmgpu_verify.argtypes = [C.c_char_p, i, i, i, d, d, d, C.c_long, d, C.c_long,
                                vp, vp, vp]
    L.lbmgpu_kernel_stats_enable.argtypes = [vp, i]
    L.lbmgpu_kernel_stats.argtypes = [vp, vp, vp, vp, i, P(i)]
    L.lbmgpu_kernel_stats_reset.argtypes = [vp]
    L.lbmgpu_kernel_timeline.argtypes = [vp, vp, vp, vp, i, P(i)]
    L.lbmgpu_launch_count.argtypes = [vp, P(C.c_long)]
    L.lbmgpu_host_alloc.argtypes = [C.c_size_t, P(vp)]
    L.lbmgpu_host_free.argtypes = [vp]
    L.lbmgpu_device_info.argtypes = [i, vp, P(i), P(C.c_size_t), P(i)]
    L.lbmgpu_synchronize.argtypes = [vp]
    L.lbmgpu_nccl_unique_id.argtypes = [vp]
    L.lbmgpu_part_info.argtypes = [vp, i, P(i), P(i), P(u64)]
    L.lbmgpu_microbench.argtypes = [C.c_char_p, u64, i, P(d)]
    L.lbmgpu_microbench_accounting.argtypes = [C.c_char_p, u64, P(u64), P(u64), P(u64)]
    L.lbmgpu_local_rows.argtypes = [vp, P(u64)]
    L.lbmgpu_local_canonical_index.argtypes = [vp, vp]
    L.lbmgpu_snapshot_local.argtypes = [vp, vp, u64]
    L.lbmgpu_load_state_local.argtypes = [vp, vp, u64]
    L.lbmgpu_halo_plan.argtypes = [i, i, i, vp, i, P(i)]
    L.lbmgpu_guard_check.argtypes = [P(i)]
    L.lbmgpu_guard_selftest.argtypes = [P(i)]
    L.lbmgpu_peer_export.argtypes = [vp, vp, C.c_size_t, P(C.c_size_t)]
    L.lbmgpu_peer_attach.argtypes = [vp, vp, C.c_size_t, i]
    L.lbmgpu_peer_probe.argtypes = [vp, i, vp, u64]
    return L


lib = _load()


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.lbmgpu_last_error().decode(errors="replace")
    if rc == 1:
        raise ConfigError(msg)
    if rc == 2:
        raise NumericalError(msg)
    raise DeviceError(msg)


# ----------------------------------------------------------------- C structs
class _Geometry(C.Structure):
    _fields_ = [("kind", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("block", C.c_int), ("spacing", C.c_int), ("pipe_diameter", C.c_int),
                ("flags", C.c_void_p), ("periodic", C.c_int * 3)]


class _Padding(C.Structure):
    _fields_ = [("mode", C.c_int), ("pads", C.c_int64 * Q)]


class _Descriptor(C.Structure):
    _fields_ = [("prop", C.c_int), ("layout_soa", C.c_int), ("indirect", C.c_int),
                ("blk", C.c_int), ("nt_streams", C.c_int), ("ria", C.c_int),
                ("pv", C.c_int), ("vec", C.c_int), ("vector_width", C.c_int)]


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int),
                ("virtual_parts", C.c_int), ("nccl_id", C.c_void_p),
                ("transport", C.c_int)]


class _VerifyReport(C.Structure):
    _fields_ = [("linf_rel", C.c_double), ("l2_rel", C.c_double),
                ("half_force_shift", C.c_double), ("steps", C.c_long),
                ("converged", C.c_int), ("passed", C.c_int)]


# -------------------------------------------------------------- model params
@dataclasses.dataclass
class TrtParams:
    """lbm::TrtParams (d3q19.hpp:64-86)."""
    omega_plus: float = 1.0
    magic_lambda: float = 3.0 / 16.0

    def viscosity(self) -> float:
        return (1.0 / self.omega_plus - 0.5) / 3.0

    def omega_minus(self) -> float:
        return lib.lbmgpu_omega_minus(self.omega_plus, self.magic_lambda)

    def validate(self) -> None:
        if not (self.omega_plus > 0.0) or not (self.omega_plus < 2.0):
            raise ConfigError(f"TrtParams: omega_plus must be in (0, 2), got {self.omega_plus}")
        if not (self.magic_lambda > 0.0):
            raise ConfigError("TrtParams: magic_lambda must be positive")

    @staticmethod
    def from_tau(tau_plus: float, lam: float = 3.0 / 16.0) -> "TrtParams":
        return TrtParams(1.0 / tau_plus, lam)


@dataclasses.dataclass
class BodyForce:
    """lbm::BodyForce (d3q19.hpp:88-92)."""
    g: Sequence[float] = (0.0, 0.0, 0.0)

    def zero(self) -> bool:
        return all(v == 0.0 for v in self.g)


# ------------------------------------------------------------------ registry
@dataclasses.dataclass
class KernelDescriptor:
    """lbm::KernelDescriptor (kernels.hpp:25-36)."""
    name: str
    prop: str = "os-push"      # os-push | os-pull | aa
    layout: str = "soa"        # soa | aos
    addr: str = "direct"       # direct | indirect
    blk: int = 0
    nt_streams: int = 0
    ria: bool = False
    pv: bool = False
    vec: bool = False
    vector_width: int = 4


_PROPS = ["os-push", "os-pull", "aa"]


def _desc_from_c(name: str, c: _Descriptor) -> KernelDescriptor:
    return KernelDescriptor(name=name, prop=_PROPS[c.prop], layout="soa" if c.layout_soa else "aos",
                            addr="indirect" if c.indirect else "direct", blk=c.blk,
                            nt_streams=c.nt_streams, ria=bool(c.ria), pv=bool(c.pv),
                            vec=bool(c.vec), vector_width=c.vector_width)


def kernel_names() -> list:
    """The 17 names in canonical reporting order (kernels.cpp:22-43)."""
    buf = C.create_string_buffer(2048)
    _check(lib.lbmgpu_kernel_names(buf, 2048))
    return buf.value.decode().split()


def is_kernel_name(name: str) -> bool:
    return name in kernel_names()


def make_descriptor(name: str, blk: int = 0, vector_width: int = 4) -> KernelDescriptor:
    """make_descriptor (kernels.cpp:50-82); ConfigError lists the valid names."""
    c = _Descriptor()
    _check(lib.lbmgpu_make_descriptor(name.encode(), blk, vector_width, C.byref(c)))
    return _desc_from_c(name, c)


def loop_balance(name: str, stats: Optional[dict] = None):
    """(reference B_l min, max, GPU algorithmic bytes per fluid update);
    stats = Kernel.ria_stats() (perfmodel.cpp:21-31: the RIA names' index
    bytes from the geometry's run count)."""
    a, b, g = C.c_double(), C.c_double(), C.c_double()
    if stats is None:
        _check(lib.lbmgpu_loop_balance(name.encode(), C.byref(a), C.byref(b), C.byref(g)))
    else:
        _check(lib.lbmgpu_loop_balance_stats(name.encode(), int(stats["total_runs"]),
                                             int(stats["n_fluid"]), C.byref(a), C.byref(b),
                                             C.byref(g)))
    return a.value, b.value, g.value


def roofline(gbps: float, bl_min: float, bl_max: float):
    """roofline (perfmodel.cpp:73-87): (P_max from the larger balance, P_max
    from the smaller one) in MFLUP/s."""
    lo, hi = C.c_double(), C.c_double()
    _check(lib.lbmgpu_roofline(float(gbps), float(bl_min), float(bl_max), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


# ------------------------------------------------------------------ geometry
KINDS = {"channel": 0, "slit": 1, "pipe": 2, "blocks": 3, "custom": 4}


@dataclasses.dataclass
class GeometrySpec:
    """lbm::GeometrySpec (geometry.hpp:36-42) + pipe_diameter extension."""
    kind: str = "channel"
    nx: int = 500
    ny: int = 100
    nz: int = 100
    block: int = 4
    spacing: int = 4
    pipe_diameter: int = 0  # 0 = reference D = min(ny, nz) - 2


@dataclasses.dataclass
class FlagField:
    """lbm::FlagField (geometry.hpp:16-29): flags in (x*ny+y)*nz+z order."""
    nx: int
    ny: int
    nz: int
    periodic: tuple
    flags: np.ndarray

    def volume(self) -> int:
        return self.nx * self.ny * self.nz

    def index(self, x, y, z) -> int:
        return (x * self.ny + y) * self.nz + z


def _geom_struct(geom):
    g = _Geometry()
    keep = None
    if isinstance(geom, FlagField):
        g.kind = 4
        g.nx, g.ny, g.nz = geom.nx, geom.ny, geom.nz
        keep = np.ascontiguousarray(geom.flags, dtype=np.uint8)
        if keep.size != geom.volume():
            raise ConfigError("FlagField: flags size does not match dims")
        g.flags = keep.ctypes.data
        for a in range(3):
            g.periodic[a] = int(bool(geom.periodic[a]))
    else:
        if geom.kind not in KINDS or geom.kind == "custom":
            raise ConfigError(f"unknown geometry kind '{geom.kind}' (valid: channel, slit, pipe, blocks)")
        g.kind = KINDS[geom.kind]
        g.nx, g.ny, g.nz = geom.nx, geom.ny, geom.nz
        g.block, g.spacing, g.pipe_diameter = geom.block, geom.spacing, geom.pipe_diameter
    return g, keep


def build_geometry(spec: GeometrySpec) -> FlagField:
    """build_geometry (geometry.cpp:40-111), generated on the device."""
    g, _keep = _geom_struct(spec)
    flags = np.zeros(spec.nx * spec.ny * spec.nz, np.uint8)
    nf = C.c_int64()
    per = (C.c_int * 3)()
    _check(lib.lbmgpu_geometry_build(C.byref(g), flags.ctypes.data, C.byref(nf), per))
    return FlagField(spec.nx, spec.ny, spec.nz, tuple(bool(p) for p in per), flags)


def fluid_count(ff: FlagField) -> int:
    return int(np.count_nonzero(ff.flags == 0))


# ------------------------------------------------------------------- padding
_PADMODES = {"none": 0, "auto": 1, "thrash": 2, "explicit": 3}


@dataclasses.dataclass
class PaddingPolicy:
    """lbm::PaddingPolicy (list_lattice.hpp:25-39)."""
    mode: str = "none"
    pads: Optional[Sequence[int]] = None

    @staticmethod
    def none():
        return PaddingPolicy("none")

    @staticmethod
    def automatic():
        return PaddingPolicy("auto")

    @staticmethod
    def thrash():
        return PaddingPolicy("thrash")

    @staticmethod
    def parse(s: str) -> "PaddingPolicy":
        """list_lattice.cpp:10-34 -- 'none' | 'auto' | 'thrash' | 19 counts."""
        if s in ("none", "auto", "thrash"):
            return PaddingPolicy(s)
        items = s.split(",")
        pads = []
        for it in items[:Q]:
            try:
                v = int(it)
            except ValueError:
                raise ConfigError(f"padding: cannot parse pad count '{it}' (example: --padding auto)")
            if v < 0:
                raise ConfigError("padding: pad counts must be >= 0")
            pads.append(v)
        if len(pads) != Q:
            raise ConfigError("padding: expected 'none', 'auto', 'thrash' or 19 comma-separated "
                              "pad counts (example: --padding auto)")
        return PaddingPolicy("explicit", pads)

    def to_string(self) -> str:
        return self.mode if self.mode != "explicit" else ",".join(str(p) for p in self.pads)

    def _c(self) -> _Padding:
        p = _Padding()
        p.mode = _PADMODES[self.mode]
        if self.pads is not None:
            for k, v in enumerate(self.pads):
                p.pads[k] = int(v)
        return p


def padding_offsets(n_fluid: int, policy: PaddingPolicy):
    """padding_offsets (list_lattice.cpp:84-121) -> (starts[19], total_slots)."""
    starts = np.zeros(Q, np.uint64)
    tot = C.c_uint64()
    p = policy._c()
    _check(lib.lbmgpu_padding_offsets(n_fluid, C.byref(p), starts.ctypes.data, C.byref(tot)))
    return starts, tot.value


# ------------------------------------------------------------- state helpers
def state_fingerprint(snapshot: np.ndarray) -> int:
    """FNV-1a over the canonical snapshot bytes (harness.cpp:27-39)."""
    a = np.ascontiguousarray(snapshot, dtype="<f8")
    return int(lib.lbmgpu_fnv1a(a.ctypes.data, a.nbytes))


_W = np.array([1.0 / 3.0] + [1.0 / 18.0] * 6 + [1.0 / 36.0] * 12)


def perturbed_equilibrium(n_fluid: int, seed: int, amplitude: float = 1e-3) -> np.ndarray:
    """perturbed_equilibrium (harness.cpp:50-62), vectorised host formula."""
    idx = np.arange(n_fluid * Q, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(seed) ^ idx
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    u01 = (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    w = np.tile(_W, n_fluid)
    return w * (1.0 + amplitude * (u01 - 0.5))


def macro_fields(snapshot: np.ndarray):
    """macro_fields (harness.cpp:64-80): bare rho and u per node."""
    f = np.asarray(snapshot, np.float64).reshape(-1, Q)
    if not np.all(np.isfinite(f)):
        raise NumericalError("macroscopic: non-finite population")
    cxs = np.array([0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0], float)
    cys = np.array([0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1], float)
    czs = np.array([0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1], float)
    rho = f.sum(axis=1)
    u = np.stack([f @ cxs, f @ cys, f @ czs], axis=1) / rho[:, None]
    return rho, u


# -------------------------------------------------------------------- kernel
@dataclasses.dataclass
class KernelCaps:
    nt_stores_available: bool = False
    nt_streams_effective: int = 0
    huge_pages_advised: bool = False


def _check_out(out, n, what):
    """The C ABI writes `n` doubles at out's data pointer: anything but a
    C-contiguous float64 array of exactly n elements would be scribbled over
    or overrun."""
    if not isinstance(out, np.ndarray) or out.dtype != np.float64:
        raise ValueError(f"{what}: out must be a float64 numpy array")
    if not out.flags.c_contiguous:
        raise ValueError(f"{what}: out must be C-contiguous")
    if out.size != n:
        raise ValueError(f"{what}: out holds {out.size} values, expected {n}")


class Kernel:
    """A GPU-resident lattice + sweep, the reference's lbm::Kernel
    (kernels.hpp:58-96).  Create with make_kernel()."""

    def __init__(self, desc: KernelDescriptor, geometry, padding: PaddingPolicy, row_pad: int = 0,
                 dist: Optional[dict] = None):
        self._h = C.c_void_p()
        g, keep = _geom_struct(geometry)
        p = padding._c()
        dp = None
        self._nccl_keep = None
        if dist:
            ds = _Dist()
            ds.rank = dist.get("rank", 0)
            ds.nranks = dist.get("nranks", 1)
            ds.device = dist.get("device", -1)
            ds.virtual_parts = dist.get("virtual_parts", 1)
            ds.transport = {"copy": 0, "peer": 1}[dist.get("transport", "copy")]
            if dist.get("nccl_id") is not None:
                self._nccl_keep = C.create_string_buffer(bytes(dist["nccl_id"]), 128)
                ds.nccl_id = C.cast(self._nccl_keep, C.c_void_p)
            dp = C.byref(ds)
        _check(lib.lbmgpu_create(desc.name.encode(), desc.blk, desc.vector_width, C.byref(g),
                                 C.byref(p), row_pad, dp, C.byref(self._h)))
        self._desc = desc
        n = C.c_uint64()
        _check(lib.lbmgpu_n_fluid(self._h, C.byref(n)))
        self._n = n.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.lbmgpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def descriptor(self) -> KernelDescriptor:
        return self._desc

    def n_fluid(self) -> int:
        return self._n

    def advance(self, params: TrtParams, force: BodyForce, steps: int) -> None:
        """Kernel::advance (kernels.cpp:84-93)."""
        g = (C.c_double * 3)(*[float(v) for v in force.g])
        _check(lib.lbmgpu_advance(self._h, params.omega_plus, params.magic_lambda, g, int(steps)))

    def time_advance(self, params: TrtParams, force: BodyForce, steps: int) -> float:
        """advance() bracketed by CUDA events on the kernel's stream; device ms."""
        g = (C.c_double * 3)(*[float(v) for v in force.g])
        ms = C.c_double()
        _check(lib.lbmgpu_time_advance(self._h, params.omega_plus, params.magic_lambda, g,
                                       int(steps), C.byref(ms)))
        return ms.value

    def snapshot(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Canonical N*19 PDFs, fluid nodes in x,y,z order.  `out`, if given,
        must be a C-contiguous float64 array of N*19 elements."""
        if out is None:
            out = np.empty(self._n * Q, np.float64)
        _check_out(out, self._n * Q, "snapshot")
        _check(lib.lbmgpu_snapshot(self._h, out.ctypes.data, out.size))
        return out

    def load_state(self, state) -> None:
        s = np.ascontiguousarray(state, np.float64)
        _check(lib.lbmgpu_load_state(self._h, s.ctypes.data, s.size))

    def run(self, state, params: TrtParams, force: BodyForce, steps: int,
            out: Optional[np.ndarray] = None):
        """load_state(state) + advance(steps) + snapshot(out) as one job
        (lbmgpu_run): bitwise the three calls; the host transfers overlap the
        sweeps when the lattice supports it and both buffers are page-locked
        (PinnedBuffer).  Returns (out, pipelined)."""
        s = np.ascontiguousarray(state, np.float64)
        if out is None:
            out = np.empty(self._n * Q, np.float64)
        _check_out(out, self._n * Q, "snapshot")
        g = (C.c_double * 3)(*[float(v) for v in force.g])
        piped = C.c_int()
        _check(lib.lbmgpu_run(self._h, params.omega_plus, params.magic_lambda, g, int(steps),
                              s.ctypes.data, s.size, out.ctypes.data, out.size, C.byref(piped)))
        return out, bool(piped.value)

    # process-local rows (split domains; == the whole state with one process)
    def local_rows(self) -> int:
        v = C.c_uint64()
        _check(lib.lbmgpu_local_rows(self._h, C.byref(v)))
        return v.value

    def local_state_size(self) -> int:
        return self.local_rows() * Q

    def local_canonical_index(self) -> np.ndarray:
        out = np.zeros(self.local_rows(), np.uint64)
        _check(lib.lbmgpu_local_canonical_index(self._h, out.ctypes.data))
        return out

    def snapshot_local(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.local_state_size(), np.float64)
        _check_out(out, self.local_state_size(), "snapshot_local")
        _check(lib.lbmgpu_snapshot_local(self._h, out.ctypes.data, out.size))
        return out

    def load_state_local(self, state) -> None:
        s = np.ascontiguousarray(state, np.float64)
        _check(lib.lbmgpu_load_state_local(self._h, s.ctypes.data, s.size))

    def load_perturbed(self, seed: int, amplitude: float = 1e-3) -> None:
        _check(lib.lbmgpu_load_perturbed(self._h, seed, amplitude))

    def total_mass(self) -> float:
        m = C.c_double()
        _check(lib.lbmgpu_total_mass(self._h, C.byref(m)))
        return m.value

    def fingerprint(self) -> int:
        v = C.c_uint64()
        _check(lib.lbmgpu_fingerprint(self._h, C.byref(v)))
        return v.value

    def capabilities(self) -> KernelCaps:
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        _check(lib.lbmgpu_capabilities(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return KernelCaps(bool(a.value), b.value, bool(c.value))

    def _ria(self):
        r, n, v, pv = C.c_int64(), C.c_int64(), C.c_double(), C.c_double()
        _check(lib.lbmgpu_ria_stats(self._h, C.byref(r), C.byref(n), C.byref(v), C.byref(pv)))
        return r.value, n.value, v.value, pv.value

    def ria_stats(self):
        r, n, _, _ = self._ria()
        return None if r < 0 else {"total_runs": r, "n_fluid": n}

    def vector_fraction(self):
        _, _, v, _ = self._ria()
        return None if v < 0 else v

    def vectorizable_fraction(self, width: int):
        """vectorizable_fraction(coding, W) (list_lattice.cpp:228-236) at any
        width; None for names without a run coding."""
        v = C.c_double()
        _check(lib.lbmgpu_vectorizable_fraction(self._h, int(width), C.byref(v)))
        return None if v.value < 0 else v.value

    def export_runs(self):
        """Run starts of the run coding in node order (run r covers
        [start[r], start[r+1]), the last up to n_fluid); None without a coding."""
        n = C.c_int64()
        _check(lib.lbmgpu_export_runs(self._h, None, 0, C.byref(n)))
        if n.value < 0:
            return None
        out = np.zeros(n.value, np.uint32)
        _check(lib.lbmgpu_export_runs(self._h, out.ctypes.data, out.size, C.byref(n)))
        return out

    def pv_chunk_fraction(self):
        _, _, _, pv = self._ria()
        return None if pv < 0 else pv

    def export_structure(self):
        """(nodes[N,3] int32, adjacency[N*18] uint32 canonical, starts[19], total)."""
        nodes = np.zeros(3 * self._n, np.int32)
        adj = np.zeros(18 * self._n, np.uint32)
        starts = np.zeros(Q, np.uint64)
        tot = C.c_uint64()
        _check(lib.lbmgpu_export_structure(self._h, nodes.ctypes.data, adj.ctypes.data,
                                           starts.ctypes.data, C.byref(tot)))
        return nodes.reshape(-1, 3), adj, starts, tot.value

    def steady_state_run(self, params, force, check_interval, rel_tol, max_steps):
        g = (C.c_double * 3)(*[float(v) for v in force.g])
        steps, conv, delta = C.c_long(), C.c_int(), C.c_double()
        _check(lib.lbmgpu_steady_state_run(self._h, params.omega_plus, params.magic_lambda, g,
                                           int(check_interval), float(rel_tol), int(max_steps),
                                           C.byref(steps), C.byref(conv), C.byref(delta)))
        return {"steps": steps.value, "converged": bool(conv.value), "final_delta": delta.value}

    # instrumentation
    def kernel_stats_enable(self, on: bool = True):
        _check(lib.lbmgpu_kernel_stats_enable(self._h, int(on)))

    def kernel_stats_reset(self):
        _check(lib.lbmgpu_kernel_stats_reset(self._h))

    def kernel_stats(self):
        cap = 32
        names = C.create_string_buffer(48 * cap)
        launches = (C.c_long * cap)()
        ms = (C.c_double * cap)()
        n = C.c_int()
        _check(lib.lbmgpu_kernel_stats(self._h, names, launches, ms, cap, C.byref(n)))
        out = {}
        for k in range(min(n.value, cap)):
            nm = names.raw[48 * k:48 * k + 48].split(b"\0", 1)[0].decode()
            out[nm] = {"launches": launches[k], "ms": ms[k]}
        return out

    def kernel_timeline(self):
        """[(name, t0_ms, t1_ms)] per recorded launch, in record order (device
        clock shared by all streams)."""
        n = C.c_int()
        _check(lib.lbmgpu_kernel_timeline(self._h, None, None, None, 0, C.byref(n)))
        cap = n.value
        if cap == 0:
            return []
        names = C.create_string_buffer(48 * cap)
        t0 = (C.c_double * cap)()
        t1 = (C.c_double * cap)()
        _check(lib.lbmgpu_kernel_timeline(self._h, names, t0, t1, cap, C.byref(n)))
        return [(names.raw[48 * k:48 * k + 48].split(b"\0", 1)[0].decode(), t0[k], t1[k])
                for k in range(min(cap, n.value))]

    def launch_count(self) -> int:
        v = C.c_long()
        _check(lib.lbmgpu_launch_count(self._h, C.byref(v)))
        return v.value

    def synchronize(self):
        _check(lib.lbmgpu_synchronize(self._h))

    def peer_export(self) -> bytes:
        """This rank's peer-transport record (CUDA IPC handles); all-gather
        the records of every rank and pass them to peer_attach()."""
        n = C.c_size_t()
        _check(lib.lbmgpu_peer_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib.lbmgpu_peer_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def peer_attach(self, records) -> None:
        """Map the neighbour slabs' lattices and flags (records in rank order)."""
        records = [bytes(r) for r in records]
        blob = b"".join(records)
        _check(lib.lbmgpu_peer_attach(self._h, blob, len(records[0]) if records else 0,
                                      len(records)))

    def peer_probe(self, which: int, plane_values: int) -> np.ndarray:
        """Boundary plane in device layout (19 x nx*ny): 0 lower neighbour's
        top plane, 1 upper neighbour's bottom plane (through the peer
        mapping), 2 own bottom plane, 3 own top plane."""
        out = np.empty(plane_values, np.float64)
        _check(lib.lbmgpu_peer_probe(self._h, which, out.ctypes.data, out.size))
        return out

    def part_info(self, part: int):
        z0, z1, nf = C.c_int(), C.c_int(), C.c_uint64()
        _check(lib.lbmgpu_part_info(self._h, part, C.byref(z0), C.byref(z1), C.byref(nf)))
        return z0.value, z1.value, nf.value


def make_kernel(desc: KernelDescriptor, geometry, padding: Optional[PaddingPolicy] = None,
                row_pad: int = 0, dist: Optional[dict] = None) -> Kernel:
    """make_kernel (kernels.hpp:102-105). `geometry` is a GeometrySpec (built
    on the device) or a host FlagField (uploaded)."""
    if padding is None:
        padding = PaddingPolicy.automatic()
    return Kernel(desc, geometry, padding, row_pad, dist)


# ------------------------------------------------------------ verification
def steady_state_run(kernel: Kernel, p: TrtParams, g: BodyForce, check_interval: int,
                     rel_tol: float, max_steps: int):
    """steady_state_run (harness.cpp:141-174) with device-side reductions."""
    return kernel.steady_state_run(p, g, check_interval, rel_tol, max_steps)


@dataclasses.dataclass
class PoiseuilleCase:
    """verification.hpp:15-22."""
    nx: int = 8
    ny: int = 8
    nz: int = 34
    g: float = 1e-6
    params: TrtParams = dataclasses.field(default_factory=lambda: TrtParams.from_tau(0.9))

    def fluid_layers(self) -> int:
        return self.nz - 2


def analytic_profile(c: PoiseuilleCase) -> np.ndarray:
    """verification.cpp:19-29."""
    h = float(c.fluid_layers())
    nu = c.params.viscosity()
    zeta = np.arange(c.fluid_layers()) + 0.5
    return c.g / (2.0 * nu) * zeta * (h - zeta)


K_VERIFY_LINF_TOLERANCE = 1e-4


def verify_kernel(k, c: PoiseuilleCase = None, check_interval: int = 200, rel_tol: float = 1e-12,
                  max_steps: int = 200000) -> dict:
    """verify_kernel (verification.cpp:31-100) on the GPU."""
    if c is None:
        c = PoiseuilleCase()
    name = k.name if isinstance(k, KernelDescriptor) else str(k)
    rep = _VerifyReport()
    layers = c.nz - 2
    sim = np.zeros(max(layers, 1))
    ana = np.zeros(max(layers, 1))
    _check(lib.lbmgpu_verify(name.encode(), c.nx, c.ny, c.nz, c.g, 1.0 / c.params.omega_plus,
                             c.params.magic_lambda, check_interval, rel_tol, max_steps,
                             C.byref(rep), sim.ctypes.data, ana.ctypes.data))
    return {"kernel": name, "dims": [c.nx, c.ny, c.nz], "g": c.g,
            "omega_plus": c.params.omega_plus, "magic_lambda": c.params.magic_lambda,
            "viscosity": c.params.viscosity(), "half_force_shift": rep.half_force_shift,
            "steps": rep.steps, "converged": bool(rep.converged),
            "simulated_ux": sim[:layers].tolist(), "analytic_ux": ana[:layers].tolist(),
            "linf_rel": rep.linf_rel, "l2_rel": rep.l2_rel,
            "tolerance": K_VERIFY_LINF_TOLERANCE, "passed": bool(rep.passed)}


# ------------------------------------------------------------------ misc
def halo_plan(nz: int, parts: int, ring: bool, one_step: bool = False):
    """z-slab halo rows (phase, src, dst, src plane, dst plane, slot0, slots):
    the AA plan (phases 0/1, z ring optional) or, one_step=True, the
    push/pull plan (phases 2/3, always with the ring)."""
    cap = 8 * parts + 8
    rows = np.zeros(7 * cap, np.int64)
    n = C.c_int()
    _check(lib.lbmgpu_halo_plan(nz, parts, 2 if one_step else int(ring), rows.ctypes.data, cap,
                                C.byref(n)))
    return rows[:7 * n.value].reshape(-1, 7)


def guard_check():
    """Debug aid: (number of live device buffers whose 4 KiB guard zones were
    overwritten, description).  Buffers get guard zones only when
    LBMGPU_GUARD=1 is set at allocation time."""
    n = C.c_int()
    rc = lib.lbmgpu_guard_check(C.byref(n))
    msg = lib.lbmgpu_last_error().decode() if n.value else ""
    _check(rc)
    return n.value, msg


def guard_selftest() -> int:
    """Negative control of guard_check (1 = the planted overrun was seen)."""
    n = C.c_int()
    _check(lib.lbmgpu_guard_selftest(C.byref(n)))
    return n.value


BOUNDARY_ROLE = ("_halo", "_peer", "peer_wait", "peer_signal", "push_halo_merge", "list_link")


def stream_overlap(timeline, boundary=BOUNDARY_ROLE):
    """Overlap evidence for the decomposed paths: of the device time the
    boundary-stream launches (boundary sweeps, peer waits / signals, halo
    merges; names containing one of `boundary`) are busy, the part during
    which an interior sweep runs at the same time.  Returns
    {"boundary_ms", "overlapped_ms", "frac"}."""
    b = [(t0, t1) for n, t0, t1 in timeline if any(x in n for x in boundary)]
    it = sorted((t0, t1) for n, t0, t1 in timeline if not any(x in n for x in boundary))
    merged = []
    for t0, t1 in it:
        if merged and t0 <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], t1)
        else:
            merged.append([t0, t1])
    busy = sum(t1 - t0 for t0, t1 in b)
    ov = 0.0
    for t0, t1 in b:
        for m0, m1 in merged:
            if m0 >= t1:
                break
            ov += max(0.0, min(t1, m1) - max(t0, m0))
    return {"boundary_ms": busy, "overlapped_ms": ov, "frac": ov / busy if busy > 0 else None}


def microbench_accounting(kind: str, working_set_bytes: int) -> dict:
    """Elements per stream and accounted bytes of one micro-benchmark pass:
    this library's (no write allocate) and the reference's
    (microbench.cpp:92-99)."""
    n, bg, br = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(lib.lbmgpu_microbench_accounting(kind.encode(), working_set_bytes, C.byref(n),
                                            C.byref(bg), C.byref(br)))
    return {"elems": n.value, "bytes_gpu": bg.value, "bytes_ref": br.value}


def microbench(kind: str, working_set_bytes: int = 8 << 30, reps: int = 5) -> float:
    """Device copy / copy-19 / copy-19-nt-sl / update-19 bandwidth in GB/s
    (reference run_microbench, microbench.cpp:57-175; GPU accounting)."""
    v = C.c_double()
    _check(lib.lbmgpu_microbench(kind.encode(), working_set_bytes, reps, C.byref(v)))
    return v.value


def micro_for(desc: KernelDescriptor) -> str:
    """Which micro-benchmark models which kernel (perfmodel.cpp:68-72)."""
    if desc.nt_streams > 0:
        return "copy-19-nt-sl"
    if desc.prop == "aa":
        return "update-19"
    return "copy-19"


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.lbmgpu_nccl_unique_id(buf))
    return buf.raw


def device_info(device: int = -1) -> dict:
    name = C.create_string_buffer(64)
    sms, l2 = C.c_int(), C.c_int()
    mem = C.c_size_t()
    _check(lib.lbmgpu_device_info(device, name, C.byref(sms), C.byref(mem), C.byref(l2)))
    return {"name": name.value.decode(), "sm_count": sms.value, "total_mem": mem.value,
            "l2_bytes": l2.value}


class PinnedBuffer:
    """Page-locked host float64 buffer (cudaMallocHost) for end-to-end runs."""

    def __init__(self, n: int):
        self._p = C.c_void_p()
        _check(lib.lbmgpu_host_alloc(n * 8, C.byref(self._p)))
        self.array = np.ctypeslib.as_array(C.cast(self._p, C.POINTER(C.c_double)), shape=(n,))

    def free(self):
        if self._p.value:
            lib.lbmgpu_host_free(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

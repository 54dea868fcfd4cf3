// Direct lattices: indexing, node decode, per-node bodies and the one-sweep kernels.
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include <type_traits>

#include "direct_args.cuh"

namespace lbmgpu {

// Element index of (storage plane, slot, y, x).  I32: 32-bit arithmetic for
// lattices of fewer than 2^32 elements (the fused L2-resident launches,
// DirectEngine::use_fused): three 32-bit multiply-adds per address instead
// of 64-bit chains.
template <bool SOA, bool I32 = false>
struct Idx {
  uint64_t P;
  uint32_t nx, ny;
  using T = std::conditional_t<I32, uint32_t, uint64_t>;
  __device__ __forceinline__ T operator()(uint32_t zs, int slot, uint32_t y, uint32_t x) const {
    if (SOA) return (T(zs) * kQ + slot) * T(P) + T(y) * nx + x;
    return ((T(zs) * ny + y) * nx + x) * kQ + slot;
  }
};

struct Coords {
  uint32_t x, y, z;        // own-plane coordinates
  uint32_t X[3], Y[3];     // wrapped x-1,x,x+1 / y-1,y,y+1
  uint32_t Z[3];           // storage planes of z-1, z, z+1
};

// own-plane coordinates -> wrapped x/y neighbours and storage planes
__device__ __forceinline__ void fill_coords(const DirectArgs& a, uint32_t x, uint32_t y,
                                            uint32_t z, Coords& c) {
  c.x = x;
  c.y = y;
  c.z = z;
  c.X[0] = x == 0 ? a.nx - 1 : x - 1;
  c.X[1] = x;
  c.X[2] = x + 1 == a.nx ? 0 : x + 1;
  c.Y[0] = y == 0 ? a.ny - 1 : y - 1;
  c.Y[1] = y;
  c.Y[2] = y + 1 == a.ny ? 0 : y + 1;
  const uint32_t zs = z + a.zoff;
  if (a.zwrap) {
    c.Z[0] = z == 0 ? a.nzl - 1 : z - 1;
    c.Z[2] = z + 1 == a.nzl ? 0 : z + 1;
  } else {
    c.Z[0] = zs - 1;
    c.Z[2] = zs + 1;
  }
  c.Z[1] = zs;
}

// own-node id n -> coordinates, wrapped x/y neighbours and storage planes
__device__ __forceinline__ void decode_node(const DirectArgs& a, uint32_t n, Coords& c) {
  const uint32_t z = a.fdP.div(n);
  const uint32_t r = n - z * a.P;
  const uint32_t y = a.fdx.div(r);
  fill_coords(a, r - y * a.nx, y, z, c);
}

__device__ __forceinline__ bool decode(const DirectArgs& a, Coords& c,
                                       uint32_t& n) {
  n = a.node0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.node0 + a.count) return false;
  if (a.band) {  // y-band order (a whole part: node0 == 0, ny % band == 0)
    const uint32_t x = n % a.nx, r = n / a.nx;
    const uint32_t per_band = a.band * a.nzl;
    const uint32_t b = r / per_band, t = r - b * per_band;
    const uint32_t z = t / a.band;
    n = (z * a.ny + b * a.band + (t - z * a.band)) * a.nx + x;
  }
  decode_node(a, n, c);
  return true;
}

// Loads of lattice data: plain (L1-cached) in the one-sweep-per-launch
// kernels; L2-only (ld.global.cg) in the fused multi-step kernel, whose later
// sweeps read lines other SMs wrote after a grid barrier.
template <bool CG>
__device__ __forceinline__ double ldp(const double* p) {
  if (CG) return __ldcg(p);
  return *p;
}
template <bool CS>
__device__ __forceinline__ void st(double* p, double v) {
  if (CS)
    __stcs(p, v);
  else
    *p = v;
}

// ---- per-node bodies (shared by the sweep kernels and the fused kernel) ----
// kernels_full_os.cpp:56-89 + full_lattice.cpp:42-56 (push, correction on dst)
template <bool SOA, bool CS, bool CG>
__device__ __forceinline__ void push_node(const DirectArgs& a, const Coords& c, uint32_t n) {
  const Idx<SOA, CG> I{a.P, a.nx, a.ny};
  double q[kQ];
  const uint32_t tm = a.tmask ? a.tmask[n] : 0u;
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = ldp<CG>(a.src + I(c.Z[1], dslot(d), c.y, c.x));
  if (!solid_node(a, c.x, c.y, c.z, n)) collide(q, a.trt);
  st<CS>(a.dst + I(c.Z[1], dslot(0), c.y, c.x), q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) {
    const uint32_t tx = c.X[1 + cx(d)], ty = c.Y[1 + cy(d)], tz = c.Z[1 + cz(d)];
    // solid target: the precomputed mask, else the neighbour's flag from L1
    // (measured faster than the arithmetic test here: cfg 1 fused 15.5k vs
    // 13.9k MFLUP/s)
    const uint32_t tn = (tz - a.zoff) * a.P + ty * a.nx + tx;
    const bool ts = a.tmask ? ((tm >> d) & 1u) != 0 : a.flags[tn] != 0;
    const int s = ts ? dslot(opp(d)) : dslot(d);
    st<CS>(a.dst + I(tz, s, ty, tx), q[d]);
  }
}

// kernels_full_os.cpp:56-89 (PULL); COLLIDE=false is the stream-only pass
template <bool SOA, bool COLLIDE, bool CS, bool CG>
__device__ __forceinline__ void pull_node(const DirectArgs& a, const Coords& c, uint32_t n) {
  const Idx<SOA, CG> I{a.P, a.nx, a.ny};
  double q[kQ];
  // Warp-uniform fast path (cf. aa_odd_node): no active lane wraps in x, y
  // or (single part) z, so the gather of direction d -- slot d of x - c_d --
  // is the own slot-0 element + odd_off[d] moved from slot opp(d) to slot d.
  // (The same form for the push's stores measured slower: cfg-5 box
  // 21.4k -> 20.2k MFLUP/s.)
  // (Not in the fused L2-resident launch (CG): there it costs registers
  // and measured 2 % slower on cfg 1.)
  constexpr bool kFast = SOA && !CG;
  const bool inner = kFast && c.x - 1u < a.nx - 2u && c.y - 1u < a.ny - 2u &&
                     (!a.zwrap || c.z - 1u < a.nzl - 2u);
  if (kFast && __all_sync(__activemask(), inner)) {
    const double* own = a.src + I(c.Z[1], 0, c.y, c.x);
    const long long P = a.P;
#pragma unroll
    for (int d = 0; d < kQ; ++d)
      q[d] = ldp<CG>(own + a.odd_off[d] + static_cast<long long>(dslot(d) - dslot(opp(d))) * P);
  } else {
    q[0] = ldp<CG>(a.src + I(c.Z[1], dslot(0), c.y, c.x));
#pragma unroll
    for (int d = 1; d < kQ; ++d)
      q[d] = ldp<CG>(a.src + I(c.Z[1 - cz(d)], dslot(d), c.Y[1 - cy(d)], c.X[1 - cx(d)]));
  }
  const bool solid = solid_node(a, c.x, c.y, c.z, n);
  if (COLLIDE && !solid) collide(q, a.trt);
  if (!COLLIDE) loads_before_stores();
  st<CS>(a.dst + I(c.Z[1], dslot(0), c.y, c.x), q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) {
    const int s = solid ? dslot(opp(d)) : dslot(d);
    st<CS>(a.dst + I(c.Z[1], s, c.y, c.x), q[d]);
  }
}

// collide_pass (kernels_full_os.cpp:149-159): fluid nodes, in place on dst
template <bool SOA, bool CG>
__device__ __forceinline__ void collide_node_pass(const DirectArgs& a, const Coords& c, uint32_t n) {
  if (solid_node(a, c.x, c.y, c.z, n)) return;
  const Idx<SOA, CG> I{a.P, a.nx, a.ny};
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = ldp<CG>(a.dst + I(c.Z[1], dslot(d), c.y, c.x));
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) a.dst[I(c.Z[1], dslot(d), c.y, c.x)] = q[d];
}

// AA pattern (kernels_full_aa.cpp:46-94), corrections dropped.  Built-in
// geometries test solidity arithmetically (no flag load ahead of the PDF
// loads; solid nodes issue no loads at all).
template <bool SOA, bool CS, bool CG>
__device__ __forceinline__ void aa_even_node(const DirectArgs& a, const Coords& c, uint32_t n) {
  if (solid_node(a, c.x, c.y, c.z, n)) return;
  const Idx<SOA, CG> I{a.P, a.nx, a.ny};
  double* buf = a.dst;
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = ldp<CG>(buf + I(c.Z[1], dslot(d), c.y, c.x));
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) st<CS>(buf + I(c.Z[1], dslot(opp(d)), c.y, c.x), q[d]);
}

template <bool SOA, bool CS, bool CG>
__device__ __forceinline__ void aa_odd_node(const DirectArgs& a, const Coords& c, uint32_t n) {
  if (solid_node(a, c.x, c.y, c.z, n)) return;
  const Idx<SOA, CG> I{a.P, a.nx, a.ny};
  double* buf = a.dst;
  // The slot direction d is gathered from, (x - c_d, opp d), is exactly the
  // slot direction opp(d) is scattered to, (x + c_opp(d), opp d): one address
  // per direction serves both the load and the store.
  double q[kQ];
  // Warp-uniform fast path: no active lane touches a wrapped neighbour, so
  // every address is the own slot-0 element plus a per-direction constant
  // (recomputed for the stores: only `own` stays live across the collision).
  const bool inner = c.x - 1u < a.nx - 2u && c.y - 1u < a.ny - 2u &&
                     (!a.zwrap || c.z - 1u < a.nzl - 2u);
  if (__all_sync(__activemask(), inner)) {
    double* own = buf + I(c.Z[1], 0, c.y, c.x);
#pragma unroll
    for (int d = 0; d < kQ; ++d) q[d] = ldp<CG>(own + a.odd_off[d]);
    collide(q, a.trt);
#pragma unroll
    for (int d = 0; d < kQ; ++d) st<CS>(own + a.odd_off[d], q[opp(d)]);
    return;
  }
  // (addresses recomputed for the stores: 19 live pointers across the
  // collision would set the kernel's register count)
  auto slot = [&](int d) {
    return buf + I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)]);
  };
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = ldp<CG>(slot(d));
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) st<CS>(slot(d), q[opp(d)]);
}

// ---- one sweep per launch, one node per thread ------------------------------
template <bool SOA, bool CS>
__global__ void __launch_bounds__(256) k_full_push(const DirectArgs a) {
  Coords c;
  uint32_t n;
  if (!decode(a, c, n)) return;
  push_node<SOA, CS, false>(a, c, n);
}

template <bool SOA, bool COLLIDE, bool CS>
__global__ void __launch_bounds__(256) k_full_pull(const DirectArgs a) {
  Coords c;
  uint32_t n;
  if (!decode(a, c, n)) return;
  pull_node<SOA, COLLIDE, CS, false>(a, c, n);
}

template <bool SOA>
__global__ void __launch_bounds__(256) k_full_collide(const DirectArgs a) {
  Coords c;
  uint32_t n;
  if (!decode(a, c, n)) return;
  collide_node_pass<SOA, false>(a, c, n);
}

// Programmatic dependent launch (the pipelined job's slab launches,
// DirectEngine::run_job): let the next grid in the stream be scheduled as
// soon as every CTA of this one runs, then wait for the previous grid to
// complete (its writes visible) before touching the lattice.  Both are
// no-ops for a launch without the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <bool SOA, bool CS, int TPB = 256, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) k_full_aa_even(const DirectArgs a) {
  pdl_enter();
  Coords c;
  uint32_t n;
  if (!decode(a, c, n)) return;
  aa_even_node<SOA, CS, false>(a, c, n);
}

template <bool SOA, bool CS, int TPB = 256, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) k_full_aa_odd(const DirectArgs a) {
  pdl_enter();
  Coords c;
  uint32_t n;
  if (!decode(a, c, n)) return;
  aa_odd_node<SOA, CS, false>(a, c, n);
}

}  // namespace lbmgpu

// Peer-memory transport of the z-slab AA decomposition:
// the odd sub-step of a slab's two boundary planes gathers from and scatters
// into the NEIGHBOUR's boundary plane directly (NVLink loads/stores through
// CUDA-IPC-mapped pointers, or plain device pointers when the slabs share one
// GPU), so no halo copy exists at all; a per-sub-step epoch flag written
// into the neighbour's memory replaces the copy's completion.
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include "direct_args.cuh"
#include "direct_node.cuh"

namespace lbmgpu {

// Which slots cross a face (kernels_full_aa.cpp:83-92 access sets, SURVEY.md
// 8(e)): the odd sub-step of node (x, y, z) reads and writes slot opp(d) of
// node x - c_d.  For the slab's bottom plane and c_z(d) = +1 that node is the
// lower neighbour's top plane (its down-slots); for the top plane and
// c_z(d) = -1 it is the upper neighbour's bottom plane (its up-slots).  The
// even sub-step touches own slots only.
struct PeerArgs {
  double* lo;         // lower neighbour's lattice (grid); null = own storage plane z-1
  double* hi;         // upper neighbour's lattice (grid); null = own storage plane z+1
  uint32_t lo_plane;  // lower neighbour's storage plane of global z0 - 1
  uint32_t hi_plane;  // upper neighbour's storage plane of global z1
  // device word set by k_peer_wait on a timeout: every later boundary sweep
  // returns before touching the neighbour's memory (a late but healthy
  // neighbour is never written out of turn)
  const int* abort;
};

__device__ __forceinline__ bool peer_aborted(const PeerArgs& pa) {
  return *static_cast<const volatile int*>(pa.abort) != 0;
}

// AA odd sub-step (kernels_full_aa.cpp:83-92, same expression as
// aa_odd_node) over boundary planes whose out-of-slab neighbours live in
// peer memory.  Each of the three z-planes a node touches has its own base
// (own lattice, or the neighbour's for the crossing plane); warps without
// an x/y wrap address every slot as base + a per-direction constant (the
// fast path of aa_odd_node).  Every thread that stored into peer memory
// ends with a system-scope fence, so its NVLink stores are visible to the
// neighbour before the kernel completes, and k_peer_signal -- the next
// launch on the stream -- publishes the epoch with a release store: the
// order is the PTX memory model's, not an assumption about kernel
// boundaries (round 1 measured such fences 1.7x slower on the
// boundary planes, ~2 % of a step at 8 slabs -- the peer transport is
// opt-in).
__global__ void __launch_bounds__(128) k_full_aa_odd_peer(const DirectArgs a, const PeerArgs pa) {
  Coords c;
  uint32_t n;
  if (peer_aborted(pa)) return;
  if (decode(a, c, n) && !solid_node(a, c.x, c.y, c.z, n)) {
    const Idx<true> I{a.P, a.nx, a.ny};
    double* zb[3] = {a.dst, a.dst, a.dst};
    uint32_t zp[3] = {c.Z[0], c.Z[1], c.Z[2]};
    if (c.z == 0 && pa.lo) {
      zb[0] = pa.lo;
      zp[0] = pa.lo_plane;
    }
    if (c.z + 1 == a.nzl && pa.hi) {
      zb[2] = pa.hi;
      zp[2] = pa.hi_plane;
    }
    double q[kQ];
    const bool inner = c.x - 1u < a.nx - 2u && c.y - 1u < a.ny - 2u;
    if (__all_sync(__activemask(), inner)) {
      // slot 0 of (plane k, y, x); direction d's slot is a constant away
      double* b[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) b[k] = zb[k] + I(zp[k], 0, c.y, c.x);
      const long long plane = static_cast<long long>(kQ) * a.P;
#pragma unroll
      for (int d = 0; d < kQ; ++d) q[d] = b[1 - cz(d)][a.odd_off[d] + cz(d) * plane];
      collide(q, a.trt);
#pragma unroll
      for (int d = 0; d < kQ; ++d) b[1 - cz(d)][a.odd_off[d] + cz(d) * plane] = q[opp(d)];
    } else {
      double* p[kQ];
      p[0] = a.dst + I(c.Z[1], dslot(0), c.y, c.x);
#pragma unroll
      for (int d = 1; d < kQ; ++d)
        p[d] = zb[1 - cz(d)] + I(zp[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)]);
#pragma unroll
      for (int d = 0; d < kQ; ++d) q[d] = p[d][0];
      collide(q, a.trt);
#pragma unroll
      for (int d = 0; d < kQ; ++d) p[d][0] = q[opp(d)];
    }
    if (zb[0] != a.dst || zb[2] != a.dst) __threadfence_system();  // crossed a face
  }
}

// One-step sweeps over z slabs with the peer transport (halo.hpp phases 2 / 3
// without the copies).  Pull (kernels_full_os.cpp:56-89, PULL): a boundary
// plane's gathers from z - 1 / z + 1 read the neighbour's source grid
// directly (remote loads only).  Push: a boundary plane's crossing stores go
// straight into the neighbour's destination grid, into slot d or -- solid
// target, from the solid-target mask built with the global flags -- the
// bounce-back slot opp(d): exactly the slot k_push_halo_merge would select,
// so the staging planes and the merge disappear.  Same arithmetic as
// pull_node / push_node.
template <bool COLLIDE>
__global__ void __launch_bounds__(256) k_full_pull_peer(const DirectArgs a, const PeerArgs pa) {
  Coords c;
  uint32_t n;
  if (peer_aborted(pa) || !decode(a, c, n)) return;
  const Idx<true> I{a.P, a.nx, a.ny};
  const double* zb[3] = {a.src, a.src, a.src};
  uint32_t zp[3] = {c.Z[0], c.Z[1], c.Z[2]};
  if (c.z == 0 && pa.lo) {
    zb[0] = pa.lo;
    zp[0] = pa.lo_plane;
  }
  if (c.z + 1 == a.nzl && pa.hi) {
    zb[2] = pa.hi;
    zp[2] = pa.hi_plane;
  }
  double q[kQ];
  q[0] = a.src[I(c.Z[1], dslot(0), c.y, c.x)];
#pragma unroll
  for (int d = 1; d < kQ; ++d)
    q[d] = zb[1 - cz(d)][I(zp[1 - cz(d)], dslot(d), c.Y[1 - cy(d)], c.X[1 - cx(d)])];
  const bool solid = solid_node(a, c.x, c.y, c.z, n);
  if (COLLIDE && !solid) collide(q, a.trt);
  if (!COLLIDE) loads_before_stores();
  a.dst[I(c.Z[1], dslot(0), c.y, c.x)] = q[0];
#pragma unroll
  for (int d = 1; d < kQ; ++d)
    a.dst[I(c.Z[1], solid ? dslot(opp(d)) : dslot(d), c.y, c.x)] = q[d];
}

__global__ void __launch_bounds__(256) k_full_push_peer(const DirectArgs a, const PeerArgs pa) {
  Coords c;
  uint32_t n;
  if (peer_aborted(pa) || !decode(a, c, n)) return;
  const Idx<true> I{a.P, a.nx, a.ny};
  const uint32_t tm = a.tmask[n];  // always built for several parts
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = a.src[I(c.Z[1], dslot(d), c.y, c.x)];
  if (!solid_node(a, c.x, c.y, c.z, n)) collide(q, a.trt);
  a.dst[I(c.Z[1], dslot(0), c.y, c.x)] = q[0];
  const bool lo = c.z == 0 && pa.lo, hi = c.z + 1 == a.nzl && pa.hi;
#pragma unroll
  for (int d = 1; d < kQ; ++d) {
    const uint32_t tx = c.X[1 + cx(d)], ty = c.Y[1 + cy(d)];
    double* base = a.dst;
    uint32_t tz = c.Z[1 + cz(d)];
    if (cz(d) < 0 && lo) {
      base = pa.lo;
      tz = pa.lo_plane;
    }
    if (cz(d) > 0 && hi) {
      base = pa.hi;
      tz = pa.hi_plane;
    }
    const int s = ((tm >> d) & 1u) ? dslot(opp(d)) : dslot(d);
    base[I(tz, s, ty, tx)] = q[d];
  }
  if (lo || hi) __threadfence_system();  // crossing stores visible before the signal (see above)
}

// Epoch flags: each part owns 4 u64 flags, [0] even done by the lower
// neighbour, [1] even done by the upper, [2] / [3] the same for odd.
// Signal: system-scope release store of `epoch` into the neighbours' flags
// (null = no neighbour on that side).
__global__ void k_peer_signal(unsigned long long* to_lo, unsigned long long* to_hi,
                              unsigned long long epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  if (to_lo) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_lo), "l"(epoch) : "memory");
  if (to_hi) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_hi), "l"(epoch) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait until the own flags f0 / f1 (null = skip) reach `epoch`.  Bounded:
// after timeout_ns the kernel records the failure in *err (host-mapped) and
// in *abort (device), and returns, so a dead neighbour cannot hang the
// device; the boundary sweeps behind it skip their peer accesses (abort)
// and the engine raises the error after the stream sync of the same
// advance() call and at every later host call (check_health).
__global__ void k_peer_wait(const unsigned long long* f0, const unsigned long long* f1,
                            unsigned long long epoch, int* err, int* abort,
                            unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  if (*static_cast<volatile int*>(abort)) return;  // already failed: no more waiting
  const unsigned long long t0 = global_ns();
  const unsigned long long* fs[2] = {f0, f1};
  for (int i = 0; i < 2; ++i) {
    if (!fs[i]) continue;
    while (ld_acquire_sys(fs[i]) < epoch) {
      if (global_ns() - t0 > timeout_ns) {
        atomicExch(abort, 1);
        atomicExch_system(err, 1);
        return;
      }
      __nanosleep(64);
    }
  }
}

}  // namespace lbmgpu

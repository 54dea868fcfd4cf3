// List lattices: kernel arguments and the sweep kernels (pull, push, collide, AA, AoS tiles).
// (part of the list-addressing translation unit, included by list.cu)
#pragma once

#include <cooperative_groups.h>

#include "lbm.hpp"
#include "tma.cuh"

namespace lbmgpu {

struct ListArgs {
  const double* src;
  double* dst;
  const uint32_t* adj;  // d-major [(d-1)*N + n]
  uint64_t N;
  uint64_t starts[kQ];  // SoA direction starts (unused for AoS)
  TrtArgs trt;
  uint64_t nb, ne;      // node range of this launch (AA sweeps); [0, N) by default
  uint64_t node_base;   // canonical sweeps over a part's local arrays: node n is local n - base
};

template <bool SOA>
__device__ __forceinline__ uint64_t lslot(const ListArgs& a, uint64_t n, int d) {
  return SOA ? a.starts[d] + (n - a.node_base) : (n - a.node_base) * kQ + d;
}

template <bool CS>
__device__ __forceinline__ void lst(double* p, double v) {
  if (CS)
    __stcs(p, v);
  else
    *p = v;
}

// PDF loads: plain in the one-sweep-per-launch kernels, L2-only
// (ld.global.cg) in the fused multi-sweep kernel, whose later sweeps read
// lines other SMs rewrote after a grid barrier.
template <bool CG>
__device__ __forceinline__ double lld(const double* p) {
  if (CG) return __ldcg(p);
  return *p;
}

// ---- per-node bodies (one-sweep kernels and the fused kernel) --------------
// list-pull (kernels_list_os.cpp:43-62, PULL)
template <bool SOA, bool COLLIDE, bool CS, bool CG>
__device__ __forceinline__ void list_pull_node(const ListArgs& a, uint64_t n) {
  uint32_t an[18];
#pragma unroll
  for (int d = 1; d < kQ; ++d) an[d - 1] = __ldg(a.adj + (d - 1) * a.N + n);
  double q[kQ];
  q[0] = lld<CG>(a.src + lslot<SOA>(a, n, 0));
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = lld<CG>(a.src + an[d - 1]);
  if (COLLIDE) collide(q, a.trt);
  if (!COLLIDE) loads_before_stores();
#pragma unroll
  for (int d = 0; d < kQ; ++d) lst<CS>(a.dst + lslot<SOA>(a, n, d), q[d]);
}

// list-push (kernels_list_os.cpp:43-62, push): own loads, scatter stores
template <bool SOA, bool CG>
__device__ __forceinline__ void list_push_node(const ListArgs& a, uint64_t n) {
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = lld<CG>(a.src + lslot<SOA>(a, n, d));
  collide(q, a.trt);
  a.dst[lslot<SOA>(a, n, 0)] = q[0];
#pragma unroll
  for (int d = 1; d < kQ; ++d) a.dst[__ldg(a.adj + (d - 1) * a.N + n)] = q[d];
}

// collide_pass (kernels_list_os.cpp:64-72), in place on dst
template <bool SOA, bool CG>
__device__ __forceinline__ void list_collide_node(const ListArgs& a, uint64_t n) {
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = lld<CG>(a.dst + lslot<SOA>(a, n, d));
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) a.dst[lslot<SOA>(a, n, d)] = q[d];
}

// aa_even_node (kernels_list_aa.cpp:10-16): own slots -> opposite slots
template <bool SOA, bool CS, bool CG>
__device__ __forceinline__ void list_aa_even_node(const ListArgs& a, uint64_t n) {
  double* buf = a.dst;
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = lld<CG>(buf + lslot<SOA>(a, n, d));
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) lst<CS>(buf + lslot<SOA>(a, n, opp(d)), q[d]);
}

// aa_odd_node (kernels_list_aa.cpp:22-31): one scatter table serves both
// sides -- gather d through column opp(d), scatter d through column d
template <bool SOA, bool CS, bool CG>
__device__ __forceinline__ void list_aa_odd_node(const ListArgs& a, uint64_t n) {
  double* buf = a.dst;
  uint32_t an[18];
#pragma unroll
  for (int d = 1; d < kQ; ++d) an[d - 1] = __ldg(a.adj + (d - 1) * a.N + n);
  double q[kQ];
  q[0] = lld<CG>(buf + lslot<SOA>(a, n, 0));
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = lld<CG>(buf + an[opp(d) - 1]);
  collide(q, a.trt);
  lst<CS>(buf + lslot<SOA>(a, n, 0), q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) lst<CS>(buf + an[d - 1], q[d]);
}

// list-pull (kernels_list_os.cpp:43-62, PULL): gather through the Gather
// table, collide, coalesced stores to own slots.  COLLIDE=false is the
// stream-only exit pass.  CS selects st.global.cs (the GPU's counterpart of
// the nt split-store variants, kernels_list_nt.cpp).
template <bool SOA, bool COLLIDE, bool CS>
__global__ void __launch_bounds__(256) k_list_pull(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  list_pull_node<SOA, COLLIDE, CS, false>(a, n);
}

// AoS list sweeps with the node's own record staged through a shared-memory
// tile of kLAosTile consecutive nodes (slots 19n + d are contiguous): full-
// sector loads / stores instead of one sector request per element.
//   k_list_aos_tile<true>:  AA even (own slots -> opposite slots), [nb, ne)
//   k_list_aos_tile<false>: collide pass, in place
//   k_list_pull_aos_tile:   pull; gathers as k_list_pull, own record stored
//                           through the tile
constexpr int kLAosTile = 128;
template <bool EVEN>
__global__ void __launch_bounds__(kLAosTile) k_list_aos_tile(const ListArgs a) {
  __shared__ __align__(128) double sh[kLAosTile * kQ];
  __shared__ __align__(8) uint64_t bar;
  const uint64_t n0 = a.nb + blockIdx.x * uint64_t(kLAosTile);
  const uint32_t cnt = static_cast<uint32_t>(min(uint64_t(kLAosTile), a.ne - n0));
  double* g = a.dst + n0 * kQ;
  aos_tile_load<kLAosTile>(sh, g, cnt, &bar);
  if (threadIdx.x < cnt) {
    double* r = sh + threadIdx.x * kQ;
    double q[kQ];
#pragma unroll
    for (int d = 0; d < kQ; ++d) q[d] = r[d];
    collide(q, a.trt);
#pragma unroll
    for (int d = 0; d < kQ; ++d) r[EVEN ? opp(d) : d] = q[d];
  }
  aos_tile_store<kLAosTile>(g, sh, cnt);
}

// Gather slot of (n, d) for an AoS list.  FROM_SCATTER: derived from the
// Scatter table the push names build (list_lattice.cpp:177-191): entry
// (n, opp d) is slot(n - c_d, opp d) when that neighbour is fluid and the
// bounce-back slot(n, d) otherwise, and the gather entry (n, d) is
// slot(n - c_d, d) resp. slot(n, opp d) -- the same record with the slot
// index d' = v % 19 replaced by opp(d') in both cases.
template <bool FROM_SCATTER>
__device__ __forceinline__ uint32_t aos_gather_slot(const ListArgs& a, uint64_t n, int d) {
  if (!FROM_SCATTER) return __ldg(a.adj + (d - 1) * a.N + n);
  const uint32_t v = __ldg(a.adj + (opp(d) - 1) * a.N + n);
  const uint32_t s = v % kQ;
  return v - s + static_cast<uint32_t>(s == 0 ? 0 : ((s & 1u) ? s + 1 : s - 1));
}

template <bool COLLIDE, bool FROM_SCATTER = false>
__global__ void __launch_bounds__(kLAosTile) k_list_pull_aos_tile(const ListArgs a) {
  __shared__ __align__(128) double sh[kLAosTile * kQ];
  const uint64_t n0 = blockIdx.x * uint64_t(kLAosTile);
  const uint32_t cnt = static_cast<uint32_t>(min(uint64_t(kLAosTile), a.N - n0));
  if (threadIdx.x < cnt) {
    const uint64_t n = n0 + threadIdx.x;
    double q[kQ];
    q[0] = a.src[n * kQ];
#pragma unroll
    for (int d = 1; d < kQ; ++d) q[d] = a.src[aos_gather_slot<FROM_SCATTER>(a, n, d)];
    if (COLLIDE) collide(q, a.trt);
    if (!COLLIDE) loads_before_stores();
    double* r = sh + threadIdx.x * kQ;
#pragma unroll
    for (int d = 0; d < kQ; ++d) r[d] = q[d];
  }
  aos_tile_store<kLAosTile>(a.dst + n0 * kQ, sh, cnt);
}

// list-push (kernels_list_os.cpp:43-62, push): own loads, scatter stores.
template <bool SOA>
__global__ void __launch_bounds__(256) k_list_push(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  list_push_node<SOA, false>(a, n);
}

// collide_pass (kernels_list_os.cpp:64-72), in place on dst.
template <bool SOA>
__global__ void __launch_bounds__(256) k_list_collide(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  list_collide_node<SOA, false>(a, n);
}

// aa_even_node (kernels_list_aa.cpp:10-16): own slots -> opposite slots.
template <bool SOA, bool CS>
__global__ void __launch_bounds__(256) k_list_aa_even(const ListArgs a) {
  const uint64_t n = a.nb + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.ne) return;
  list_aa_even_node<SOA, CS, false>(a, n);
}

// aa_odd_node (kernels_list_aa.cpp:22-31): one scatter table serves both
// sides -- gather d through column opp(d), scatter d through column d.
template <bool SOA, bool CS>
__global__ void __launch_bounds__(256) k_list_aa_odd(const ListArgs a, uint64_t pf) {
  const uint64_t n = a.nb + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.ne) return;
  double* buf = a.dst;
  // L2 prefetch of the adjacency lines a block about `pf` nodes ahead will
  // need (blocks are dispatched in index order): the index load of later
  // blocks then hits L2 and the index -> gather chain shortens.  Lanes 0..17
  // of each warp each touch one 128 B column line of that warp.
  if (pf) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t m = (n & ~uint64_t(31)) + pf;
    if (lane < 18 && m < a.N)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.adj + lane * a.N + m));
  }
  (void)buf;
  list_aa_odd_node<SOA, CS, false>(a, n);
}

// ---- fused multi-sweep launch for L2-resident list lattices ---------------
// As k_full_fused (direct_fused.cuh): one cooperative launch runs all sweeps,
// cooperative-groups grid sync between them, grid-stride node loops, PDF
// loads ld.global.cg, the per-node bodies above -- bitwise the per-sweep
// kernels' results.
enum ListFusedKind { kListFusedAA = 0, kListFusedPush = 1, kListFusedPull = 2 };
template <bool SOA, int KIND, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_list_fused(ListArgs a, double* other, long sweeps) {
  const uint64_t G = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t i0 = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  double* bufs[2] = {a.dst, other};
  for (long s = 0; s < sweeps; ++s) {
    if (KIND == kListFusedAA) {
      for (uint64_t n = i0; n < a.N; n += G)
        (s & 1) ? list_aa_odd_node<SOA, false, true>(a, n)
                : list_aa_even_node<SOA, false, true>(a, n);
    } else if (KIND == kListFusedPush) {
      a.src = bufs[s & 1];
      a.dst = bufs[(s & 1) ^ 1];
      for (uint64_t n = i0; n < a.N; n += G) list_push_node<SOA, true>(a, n);
    } else if (s == 0) {  // pull: collide pass on the current grid
      a.dst = bufs[0];
      for (uint64_t n = i0; n < a.N; n += G) list_collide_node<SOA, true>(a, n);
    } else {
      a.src = bufs[(s - 1) & 1];
      a.dst = bufs[s & 1];
      if (s + 1 < sweeps)
        for (uint64_t n = i0; n < a.N; n += G) list_pull_node<SOA, true, false, true>(a, n);
      else
        for (uint64_t n = i0; n < a.N; n += G) list_pull_node<SOA, false, false, true>(a, n);
    }
    if (s + 1 < sweeps) grid.sync();
  }
}

}  // namespace lbmgpu

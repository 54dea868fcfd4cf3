// Indirect (list / adjacency) addressing: list-push-*, list-pull-*,
// list-pull-split-nt-*, list-aa-*, list-aa-ria-soa, list-aa-pv-soa.
//
// Reference: ListLattice / build_structure (src/list_lattice.cpp:123-310),
// ListOsKernel (src/kernels_list_os.cpp:9-97), ListNtKernel
// (src/kernels_list_nt.cpp:77-167), ListAaKernel / ListAaRiaKernel
// (src/kernels_list_aa.cpp:8-251).
//
// The structure is built ON THE DEVICE and is bit-exact with the reference:
//  * node order (order_nodes, :123-141): a bijective traversal position t(i)
//    per box node (blk = 0: canonical x,y,z; blk > 0: the y-z tile order),
//    an exclusive scan of the fluid flags in t order gives the list rank;
//  * SoA slot map: starts[d] + n with the reference's padding_offsets;
//    AoS: 19n + d (list_lattice.hpp:66-75);
//  * adjacency entry (n, d) (:177-191): neighbour at n + c_look (look = d for
//    Scatter, opp(d) for Gather; periodic wrap, else Outside) -> slot(m, d)
//    if fluid else slot(n, opp d) (half-way bounce-back baked in).
// The PDF arrays keep the reference slot numbering exactly (the adjacency
// values ARE slot numbers); only the adjacency ARRAY is stored d-major,
// adj[(d-1)*N + n], so the 18 index loads of a warp are coalesced.  The
// canonical [n*18 + d-1] order is produced on export.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "lbm.hpp"

namespace lbmgpu {

struct ListArgs {
  const double* src;
  double* dst;
  const uint32_t* adj;  // d-major [(d-1)*N + n]
  uint64_t N;
  uint64_t starts[kQ];  // SoA direction starts (unused for AoS)
  TrtArgs trt;
};

template <bool SOA>
__device__ __forceinline__ uint64_t lslot(const ListArgs& a, uint64_t n, int d) {
  return SOA ? a.starts[d] + n : n * kQ + d;
}

template <bool CS>
__device__ __forceinline__ void lst(double* p, double v) {
  if (CS)
    __stcs(p, v);
  else
    *p = v;
}

// list-pull (kernels_list_os.cpp:43-62, PULL): gather through the Gather
// table, collide, coalesced stores to own slots.  COLLIDE=false is the
// stream-only exit pass.  CS selects st.global.cs (the GPU's counterpart of
// the nt split-store variants, kernels_list_nt.cpp).
template <bool SOA, bool COLLIDE, bool CS>
__global__ void __launch_bounds__(256) k_list_pull(const ListArgs a, uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  if (pf) {  // adjacency L2 prefetch for a later wave (see k_list_aa_odd)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t m = (n & ~uint64_t(31)) + pf;
    if (lane < 18 && m < a.N)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.adj + lane * a.N + m));
  }
  uint32_t an[18];
#pragma unroll
  for (int d = 1; d < kQ; ++d) an[d - 1] = __ldg(a.adj + (d - 1) * a.N + n);
  double q[kQ];
  q[0] = a.src[lslot<SOA>(a, n, 0)];
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = a.src[an[d - 1]];
  if (COLLIDE) collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) lst<CS>(a.dst + lslot<SOA>(a, n, d), q[d]);
}

// list-push (kernels_list_os.cpp:43-62, push): own loads, scatter stores.
template <bool SOA>
__global__ void __launch_bounds__(256) k_list_push(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = a.src[lslot<SOA>(a, n, d)];
  collide(q, a.trt);
  a.dst[lslot<SOA>(a, n, 0)] = q[0];
#pragma unroll
  for (int d = 1; d < kQ; ++d) a.dst[__ldg(a.adj + (d - 1) * a.N + n)] = q[d];
}

// collide_pass (kernels_list_os.cpp:64-72), in place on dst.
template <bool SOA>
__global__ void __launch_bounds__(256) k_list_collide(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = a.dst[lslot<SOA>(a, n, d)];
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) a.dst[lslot<SOA>(a, n, d)] = q[d];
}

// aa_even_node (kernels_list_aa.cpp:10-16): own slots -> opposite slots.
template <bool SOA, bool CS>
__global__ void __launch_bounds__(256) k_list_aa_even(const ListArgs a) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  double* buf = a.dst;
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) q[d] = buf[lslot<SOA>(a, n, d)];
  collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) lst<CS>(buf + lslot<SOA>(a, n, opp(d)), q[d]);
}

// aa_odd_node (kernels_list_aa.cpp:22-31): one scatter table serves both
// sides -- gather d through column opp(d), scatter d through column d.
template <bool SOA, bool CS>
__global__ void __launch_bounds__(256) k_list_aa_odd(const ListArgs a, uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
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
  uint32_t an[18];
#pragma unroll
  for (int d = 1; d < kQ; ++d) an[d - 1] = __ldg(a.adj + (d - 1) * a.N + n);
  double q[kQ];
  q[0] = buf[lslot<SOA>(a, n, 0)];
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = buf[an[opp(d) - 1]];
  collide(q, a.trt);
  lst<CS>(buf + lslot<SOA>(a, n, 0), q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) lst<CS>(buf + an[d - 1], q[d]);
}

// Persistent variant of k_list_aa_odd: every thread walks n, n+G, ... and
// loads the 18 adjacency entries of its NEXT node while the current node's
// gathers and collision are in flight, so the index-load latency no longer
// sits in series in front of the dependent PDF gathers.
template <bool SOA>
__global__ void __launch_bounds__(256, 2) k_list_aa_odd_pipe(const ListArgs a) {
  const uint64_t G = uint64_t(gridDim.x) * blockDim.x;
  uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  double* buf = a.dst;
  uint32_t an[18];
  if (n < a.N) {
#pragma unroll
    for (int d = 1; d < kQ; ++d) an[d - 1] = __ldg(a.adj + (d - 1) * a.N + n);
  }
  for (; n < a.N; n += G) {
    double q[kQ];
    q[0] = buf[lslot<SOA>(a, n, 0)];
#pragma unroll
    for (int d = 1; d < kQ; ++d) q[d] = buf[an[opp(d) - 1]];
    uint32_t nx[18];
    const uint64_t m = n + G;
    if (m < a.N) {
#pragma unroll
      for (int d = 1; d < kQ; ++d) nx[d - 1] = __ldg(a.adj + (d - 1) * a.N + m);
    }
    collide(q, a.trt);
    buf[lslot<SOA>(a, n, 0)] = q[0];
#pragma unroll
    for (int d = 1; d < kQ; ++d) buf[an[d - 1]] = q[d];
#pragma unroll
    for (int d = 0; d < 18; ++d) an[d] = nx[d];
  }
}

// ---- structure construction -------------------------------------------------
// Traversal position of box node (x,y,z) in order_nodes (list_lattice.cpp:
// 127-140).  blk > 0: tiles (ty, tz) in row-major order, inside a tile x, then
// y, then z; the tile at (ty, tz) with extents th x tw starts after
// nx*(ty*nz + th*tz) positions.
__device__ __forceinline__ uint64_t trav_pos(int x, int y, int z, int nx,
                                             int ny, int nz, int blk) {
  if (blk == 0) return (uint64_t(x) * ny + y) * nz + z;
  const int ty = y / blk * blk, tz = z / blk * blk;
  const int th = min(blk, ny - ty), tw = min(blk, nz - tz);
  return uint64_t(nx) * (uint64_t(ty) * nz + uint64_t(th) * tz) +
         uint64_t(x) * th * tw + uint64_t(y - ty) * tw + (z - tz);
}

__global__ void k_trav_flags(const uint8_t* __restrict__ flags, int nx, int ny,
                             int nz, int blk, uint8_t* __restrict__ ft) {
  const uint64_t V = uint64_t(nx) * ny * nz;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < V;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int z = static_cast<int>(i % nz);
    const uint64_t r = i / nz;
    const int y = static_cast<int>(r % ny), x = static_cast<int>(r / ny);
    ft[trav_pos(x, y, z, nx, ny, nz, blk)] = flags[i];
  }
}

// rank (list_lattice.cpp:160-164), nodes, canonical <-> list maps.
__global__ void k_rank_nodes(const uint8_t* __restrict__ flags,
                             const uint32_t* __restrict__ trank,
                             const uint32_t* __restrict__ crank, int nx, int ny,
                             int nz, int blk, uint32_t* __restrict__ rank,
                             int32_t* __restrict__ nodes,
                             uint32_t* __restrict__ list_of_canon) {
  const uint64_t V = uint64_t(nx) * ny * nz;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < V;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (flags[i]) {
      rank[i] = 0xffffffffu;
      continue;
    }
    const int z = static_cast<int>(i % nz);
    const uint64_t r = i / nz;
    const int y = static_cast<int>(r % ny), x = static_cast<int>(r / ny);
    const uint32_t n = blk == 0 ? crank[i] : trank[trav_pos(x, y, z, nx, ny, nz, blk)];
    rank[i] = n;
    nodes[3 * uint64_t(n)] = x;
    nodes[3 * uint64_t(n) + 1] = y;
    nodes[3 * uint64_t(n) + 2] = z;
    if (list_of_canon) list_of_canon[crank[i]] = n;
  }
}

struct AdjBuild {
  const uint8_t* flags;
  const uint32_t* rank;
  const int32_t* nodes;
  uint32_t* adj;  // d-major
  uint64_t N;
  int nx, ny, nz;
  int per[3];
  int soa, scatter;
  uint64_t starts[kQ];
};

// build_structure adjacency loop (list_lattice.cpp:177-191) with the
// neighbor() rule (geometry.cpp:119-131).
__global__ void k_build_adj(const AdjBuild b) {
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < b.N;
       n += uint64_t(gridDim.x) * blockDim.x) {
    const int x = b.nodes[3 * n], y = b.nodes[3 * n + 1], z = b.nodes[3 * n + 2];
#pragma unroll
    for (int d = 1; d < kQ; ++d) {
      const int look = b.scatter ? d : opp(d);
      int t0 = x + cx(look), t1 = y + cy(look), t2 = z + cz(look);
      bool outside = false;
      if (t0 < 0 || t0 >= b.nx) {
        if (!b.per[0]) outside = true; else t0 = (t0 + b.nx) % b.nx;
      }
      if (!outside && (t1 < 0 || t1 >= b.ny)) {
        if (!b.per[1]) outside = true; else t1 = (t1 + b.ny) % b.ny;
      }
      if (!outside && (t2 < 0 || t2 >= b.nz)) {
        if (!b.per[2]) outside = true; else t2 = (t2 + b.nz) % b.nz;
      }
      uint64_t slot;
      const uint64_t ti = (uint64_t(t0) * b.ny + t1) * b.nz + t2;
      if (!outside && b.flags[ti] == 0) {
        const uint64_t m = b.rank[ti];
        slot = b.soa ? b.starts[d] + m : m * kQ + d;
      } else {
        slot = b.soa ? b.starts[opp(d)] + n : n * kQ + opp(d);
      }
      b.adj[(d - 1) * b.N + n] = static_cast<uint32_t>(slot);
    }
  }
}

__global__ void k_adj_canonical(const uint32_t* __restrict__ adj, uint64_t N,
                                uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < N * 18;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t n = i / 18;
    const int dm1 = static_cast<int>(i - n * 18);
    out[i] = adj[dm1 * N + n];
  }
}

// RIA run starts (build_ria, list_lattice.cpp:206-226): node n starts a run
// if n == 0 or its pattern of 18 relative offsets differs from node n-1's.
__global__ void k_ria_starts(const uint32_t* __restrict__ adj, uint64_t N,
                             int soa, const ListArgs a,
                             uint8_t* __restrict__ is_start) {
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < N;
       n += uint64_t(gridDim.x) * blockDim.x) {
    bool start = n == 0;
    if (!start)
      for (int d = 1; d < kQ && !start; ++d) {
        const uint64_t sn = soa ? a.starts[d] + n : n * kQ + d;
        const uint64_t sp = soa ? a.starts[d] + n - 1 : (n - 1) * kQ + d;
        const int32_t pn = static_cast<int32_t>(int64_t(adj[(d - 1) * N + n]) - int64_t(sn));
        const int32_t pp = static_cast<int32_t>(int64_t(adj[(d - 1) * N + n - 1]) - int64_t(sp));
        start = pn != pp;
      }
    is_start[n] = start;
  }
}

// ---- RIA: run-coded odd step (list-aa-ria-soa / list-aa-pv-soa) -------------
struct IsStart {
  __host__ __device__ __forceinline__ uint32_t operator()(uint8_t f) const { return f; }
};

// The reference (kernels_list_aa.cpp:185-224) walks runs of consecutive nodes
// that share one pattern of 18 relative offsets (entry - own slot) and
// resolves the slot bases once per run.  GPU form: the run of node n is found
// from a per-32-node table (first run id + a bitmask of run starts, 8 B per
// 32 nodes) and the run's 18 offsets are read from a small pattern table that
// stays in L1/L2 (warps mostly share one run).  Index traffic drops from
// 72 B per odd update to ~0.25 B + the amortised pattern rows; results are
// bitwise those of list-aa-soa (same loads, same collide, same stores).
__global__ void k_ria_tables(const uint8_t* __restrict__ is_start,
                             const uint32_t* __restrict__ run_incl, uint64_t N,
                             uint32_t* __restrict__ run_start,
                             uint32_t* __restrict__ warp_run0,
                             uint32_t* __restrict__ warp_mask) {
  // launched with blockDim a multiple of 32 and N padded to whole warps
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const bool valid = n < N;
  const bool st = valid && is_start[n];
  const uint32_t r = valid ? run_incl[n] - 1 : 0;
  if (st) run_start[r] = static_cast<uint32_t>(n);
  const uint32_t mask = __ballot_sync(0xffffffffu, st);
  if ((threadIdx.x & 31) == 0 && valid) {
    warp_run0[n >> 5] = r;
    warp_mask[n >> 5] = mask;
  }
}

__global__ void k_ria_patterns(const uint32_t* __restrict__ adj,
                               const uint32_t* __restrict__ run_start, uint64_t R,
                               const ListArgs a, int32_t* __restrict__ pat) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R * 18;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / 18;
    const int d = static_cast<int>(i - r * 18) + 1;
    const uint64_t s = run_start[r];
    pat[i] = static_cast<int32_t>(int64_t(adj[(d - 1) * a.N + s]) -
                                  int64_t(a.starts[d] + s));
  }
}

template <bool CS>
__global__ void __launch_bounds__(256) k_list_aa_odd_ria(const ListArgs a,
                                                         const int32_t* __restrict__ pat,
                                                         const uint32_t* __restrict__ warp_run0,
                                                         const uint32_t* __restrict__ warp_mask,
                                                         uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  const uint32_t lane = threadIdx.x & 31;
  if (pf && lane == 0) {  // L2 prefetch of a later wave's run-table words
    const uint64_t w = (n >> 5) + pf / 32;
    if (w * 32 < a.N) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(warp_run0 + w));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(warp_mask + w));
    }
  }
  const uint32_t below = (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u)) & ~1u;
  const uint32_t r = __ldg(warp_run0 + (n >> 5)) + __popc(__ldg(warp_mask + (n >> 5)) & below);
  const int32_t* p = pat + uint64_t(r) * 18;
  double* buf = a.dst;
  // entry(n, k) = starts[k] + n + pattern[k-1]  (list_lattice.cpp:206-226)
  int64_t off[18];
#pragma unroll
  for (int k = 0; k < 18; ++k) off[k] = __ldg(p + k);
  double q[kQ];
  q[0] = buf[a.starts[0] + n];
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = buf[int64_t(a.starts[opp(d)] + n) + off[opp(d) - 1]];
  collide(q, a.trt);
  lst<CS>(buf + a.starts[0] + n, q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) lst<CS>(buf + int64_t(a.starts[d] + n) + off[d - 1], q[d]);
}

// Group-pattern form of the run coding: a 32-node group (one warp) that lies
// inside a single run carries that run's 18 offsets inline (72 B per 32
// nodes, loaded as warp broadcasts with no dependent lookup in front); a
// group that straddles run boundaries is marked (first offset = INT32_MIN)
// and its nodes read their own scatter-table entries.  Same loads, collide
// and stores as list-aa-soa, so bitwise identical.
constexpr int32_t kMixedGroup = INT32_MIN;

__global__ void k_ria_group_patterns(const int32_t* __restrict__ pat,
                                     const uint32_t* __restrict__ warp_run0,
                                     const uint32_t* __restrict__ warp_mask, uint64_t N,
                                     int32_t* __restrict__ gpat) {
  const uint64_t groups = (N + 31) / 32;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < groups * 18;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g = i / 18;
    const int k = static_cast<int>(i - g * 18);
    const bool full = (g + 1) * 32 <= N;
    const bool uniform = full && (warp_mask[g] & ~1u) == 0;
    gpat[i] = uniform ? pat[uint64_t(warp_run0[g]) * 18 + k] : (k == 0 ? kMixedGroup : 0);
  }
}

template <bool CS>
__global__ void __launch_bounds__(256) k_list_aa_odd_gpat(const ListArgs a,
                                                          const int32_t* __restrict__ gpat,
                                                          uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  if (pf) {  // L2 prefetch of the group row a later wave needs (see k_list_aa_odd)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t g = (n >> 5) + pf / 32;
    if (lane < 2 && g * 32 < a.N)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(gpat + g * 18 + lane * 16));
  }
  const int32_t* row = gpat + (n >> 5) * 18;
  double* buf = a.dst;
  int64_t ent[18];  // scatter-table entries of node n
  const int32_t first = __ldg(row);
  if (first != kMixedGroup) {
    // entry(n, k) = starts[k] + n + pattern[k-1]  (list_lattice.cpp:206-226)
    ent[0] = int64_t(a.starts[1] + n) + first;
#pragma unroll
    for (int k = 1; k < 18; ++k) ent[k] = int64_t(a.starts[k + 1] + n) + __ldg(row + k);
  } else {
#pragma unroll
    for (int k = 0; k < 18; ++k) ent[k] = __ldg(a.adj + uint64_t(k) * a.N + n);
  }
  double q[kQ];
  q[0] = buf[a.starts[0] + n];
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = buf[ent[opp(d) - 1]];
  collide(q, a.trt);
  lst<CS>(buf + a.starts[0] + n, q[0]);
#pragma unroll
  for (int d = 1; d < kQ; ++d) lst<CS>(buf + ent[d - 1], q[d]);
}

template <bool SOA>
__global__ void k_list_init(double* buf, const ListArgs a) {
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < a.N;
       n += uint64_t(gridDim.x) * blockDim.x)
#pragma unroll
    for (int d = 0; d < kQ; ++d) buf[lslot<SOA>(a, n, d)] = weight(d);
}

// canonical gather / scatter / perturbation / macro fields over c in
// [c0, c1): list node n = list_of_canon[c] (identity for blk = 0).
template <bool SOA, int MODE>  // 0 gather, 1 scatter, 2 perturb, 3 macro
__global__ void k_list_canon(const ListArgs a, double* buf,
                             const uint32_t* __restrict__ loc, uint64_t c0,
                             uint64_t c1, double* stage, uint64_t seed,
                             double amp, double* rho, double* u) {
  for (uint64_t c = c0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
       c < c1; c += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t n = loc ? loc[c] : c;
    if (MODE == 0) {
#pragma unroll
      for (int d = 0; d < kQ; ++d) stage[(c - c0) * kQ + d] = buf[lslot<SOA>(a, n, d)];
    } else if (MODE == 1) {
#pragma unroll
      for (int d = 0; d < kQ; ++d) buf[lslot<SOA>(a, n, d)] = stage[(c - c0) * kQ + d];
    } else if (MODE == 2) {
#pragma unroll
      for (int d = 0; d < kQ; ++d)
        buf[lslot<SOA>(a, n, d)] = perturbed_value(c, d, seed, amp);
    } else {
      double f[kQ];
#pragma unroll
      for (int d = 0; d < kQ; ++d) f[d] = buf[lslot<SOA>(a, n, d)];
      double r, ux, uy, uz;
      macroscopic(f, r, ux, uy, uz);
      rho[c] = r;
      u[3 * c] = ux;
      u[3 * c + 1] = uy;
      u[3 * c + 2] = uz;
    }
  }
}

template <bool SOA>
__global__ void k_list_mass_terms(const ListArgs a, const double* buf,
                                  double* out) {
  // contiguous copy of the fluid populations (pads excluded) for the
  // compensated sum
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < a.N;
       n += uint64_t(gridDim.x) * blockDim.x)
#pragma unroll
    for (int d = 0; d < kQ; ++d) out[d * a.N + n] = buf[lslot<SOA>(a, n, d)];
}

// ------------------------------------------------------------------ engine
namespace {

int grid_for(uint64_t n, int threads) {
  return static_cast<int>(std::min<uint64_t>(ceil_div(n, threads), 148ull * 64));
}

class ListEngine final : public Engine {
 public:
  ListEngine(const Descriptor& d, const GeomSpec& g, const Padding& pad) {
    desc_ = d;
    LBM_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    DeviceGeometry geo = build_geometry_device(g, stream_);
    nx_ = geo.nx;
    ny_ = geo.ny;
    nz_ = geo.nz;
    per_ = geo.periodic;
    const uint64_t V = geo.volume();
    n_fluid_ = static_cast<uint64_t>(geo.n_fluid);
    if (n_fluid_ >= (1ull << 32))
      throw ConfigError("list lattice: more than 2^32 fluid nodes");

    // slot map (list_lattice.cpp:166-173)
    uint64_t total = 0;
    std::array<uint64_t, kQ> st{};
    if (d.soa) {
      st = padding_offsets(n_fluid_, pad, &total);
    } else {
      total = n_fluid_ * kQ;
    }
    if (total >= (1ull << 32))
      throw ConfigError("list lattice: " + std::to_string(total) +
                        " PDF slots exceed the 32-bit adjacency range");
    total_slots_ = total;
    for (int q = 0; q < kQ; ++q) starts_[q] = st[q];

    // ranks in traversal order and canonical order
    DevBuf<uint32_t> crank(V);
    scan_fluid(geo.flags.get(), crank.get(), V, stream_);
    DevBuf<uint32_t> trank;
    if (d.blk > 0) {
      DevBuf<uint8_t> ft(V);
      k_trav_flags<<<grid_for(V, 256), 256, 0, stream_>>>(geo.flags.get(), nx_,
                                                          ny_, nz_, d.blk,
                                                          ft.get());
      LBM_CHECK_LAUNCH();
      trank.alloc(V);
      scan_fluid(ft.get(), trank.get(), V, stream_);
      list_of_canon_.alloc(n_fluid_);
    }
    DevBuf<uint32_t> rank(V);
    nodes_.alloc(3 * n_fluid_);
    k_rank_nodes<<<grid_for(V, 256), 256, 0, stream_>>>(
        geo.flags.get(), trank.get(), crank.get(), nx_, ny_, nz_, d.blk,
        rank.get(), nodes_.get(), d.blk > 0 ? list_of_canon_.get() : nullptr);
    LBM_CHECK_LAUNCH();

    // adjacency: Gather for pull, Scatter for push and AA
    // (kernels_list_os.cpp:19-20, kernels_list_aa.cpp:40)
    scatter_ = d.prop != Prop::OsPull;
    adj_.alloc(18 * n_fluid_);
    AdjBuild b{};
    b.flags = geo.flags.get();
    b.rank = rank.get();
    b.nodes = nodes_.get();
    b.adj = adj_.get();
    b.N = n_fluid_;
    b.nx = nx_;
    b.ny = ny_;
    b.nz = nz_;
    for (int a = 0; a < 3; ++a) b.per[a] = per_[a];
    b.soa = d.soa;
    b.scatter = scatter_;
    for (int q = 0; q < kQ; ++q) b.starts[q] = starts_[q];
    k_build_adj<<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(b);
    LBM_CHECK_LAUNCH();

    // PDF buffers initialised to the weights (list_lattice.cpp:248-264);
    // pad slots are zeroed (the reference leaves them untouched).
    const int nbuf = d.prop == Prop::Aa ? 1 : 2;
    for (int q = 0; q < nbuf; ++q) {
      buf_[q].alloc(total_slots_);
      LBM_CUDA(cudaMemsetAsync(buf_[q].get(), 0, buf_[q].bytes(), stream_));
      ListArgs a = base_args();
      d.soa ? k_list_init<true><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(buf_[q].get(), a)
            : k_list_init<false><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(buf_[q].get(), a);
      LBM_CHECK_LAUNCH();
    }
    LBM_CUDA(cudaStreamSynchronize(stream_));
    // streaming stores for the nt names and for lattices far beyond L2
    cs_nt_ = d.nt_streams > 0;
    if (d.ria) build_ria();
    {
      int dev = 0;
      LBM_CUDA(cudaGetDevice(&dev));
      LBM_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev));
      if (const char* e = std::getenv("LBMGPU_LIST_ODD_PIPE")) odd_pipe_ = std::atoi(e) != 0;
      if (const char* e = std::getenv("LBMGPU_RIA_MODE")) ria_mode_ = std::atoi(e);
      // adjacency L2 prefetch distance, in resident-grid waves (0 = off)
      int waves = 1;  // measured best on B200 (cfg 2 list-aa odd: 5946 -> 6530 GB/s)
      if (const char* e = std::getenv("LBMGPU_LIST_PF_WAVES")) waves = std::atoi(e);
      pf_ = uint64_t(waves) * uint64_t(sm_count_) * 2 * 256;
      int pwaves = 0;
      if (const char* e = std::getenv("LBMGPU_PULL_PF_WAVES")) pwaves = std::atoi(e);
      pull_pf_ = uint64_t(pwaves) * uint64_t(sm_count_) * 2 * 256;
    }
  }

  ~ListEngine() override {
    if (stream_) cudaStreamDestroy(stream_);
  }

  ListArgs base_args() const {
    ListArgs a{};
    a.adj = adj_.get();
    a.N = n_fluid_;
    for (int q = 0; q < kQ; ++q) a.starts[q] = starts_[q];
    return a;
  }

  template <class K, class... Extra>
  void launch(const char* name, K kern, const ListArgs& a, Extra... extra) {
    const int threads = 256;
    const int tok = stats_.begin(name, stream_);
    kern<<<static_cast<unsigned>(ceil_div(a.N, threads)), threads, 0, stream_>>>(a, extra...);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  void advance(const TrtArgs& t, long steps) override {
    ListArgs a = base_args();
    a.trt = t;
    const bool soa = desc_.soa;
    if (desc_.prop == Prop::Aa) {
      a.src = a.dst = buf_[0].get();
      for (long s = 0; s < steps; s += 2) {
        soa ? launch("list_aa_even_soa", k_list_aa_even<true, false>, a)
            : launch("list_aa_even_aos", k_list_aa_even<false, false>, a);
        if (desc_.ria && soa) {
          const int tok = stats_.begin("list_aa_odd_ria_soa", stream_);
          const unsigned g = static_cast<unsigned>(ceil_div(a.N, 256));
          if (ria_mode_ == 1)
            k_list_aa_odd_gpat<false><<<g, 256, 0, stream_>>>(a, ria_gpat_.get(), pf_);
          else
            k_list_aa_odd_ria<false><<<g, 256, 0, stream_>>>(a, ria_pat_.get(), ria_run0_.get(),
                                                             ria_mask_.get(), pf_);
          LBM_CHECK_LAUNCH();
          stats_.end(tok, stream_);
        } else if (odd_pipe_) {
          const int tok = stats_.begin(soa ? "list_aa_odd_soa" : "list_aa_odd_aos", stream_);
          const unsigned grid = static_cast<unsigned>(
              std::min<uint64_t>(ceil_div(a.N, 256), uint64_t(sm_count_) * 2));
          if (soa)
            k_list_aa_odd_pipe<true><<<grid, 256, 0, stream_>>>(a);
          else
            k_list_aa_odd_pipe<false><<<grid, 256, 0, stream_>>>(a);
          LBM_CHECK_LAUNCH();
          stats_.end(tok, stream_);
        } else {
          soa ? launch("list_aa_odd_soa", k_list_aa_odd<true, false>, a, pf_)
              : launch("list_aa_odd_aos", k_list_aa_odd<false, false>, a, pf_);
        }
      }
      return;
    }
    if (desc_.prop == Prop::OsPush) {
      for (long s = 0; s < steps; ++s) {
        a.src = buf_[cur_].get();
        a.dst = buf_[1 - cur_].get();
        soa ? launch("list_push_soa", k_list_push<true>, a)
            : launch("list_push_aos", k_list_push<false>, a);
        cur_ ^= 1;
      }
      return;
    }
    // pull: collide pass, T-1 fused sweeps, one stream-only sweep
    // (kernels_list_os.cpp:74-91, kernels_list_nt.cpp:146-158)
    a.src = a.dst = buf_[cur_].get();
    soa ? launch("list_collide_soa", k_list_collide<true>, a)
        : launch("list_collide_aos", k_list_collide<false>, a);
    for (long s = 0; s < steps; ++s) {
      a.src = buf_[cur_].get();
      a.dst = buf_[1 - cur_].get();
      const bool last = s == steps - 1;
      if (soa) {
        if (last)
          launch("list_pull_stream_soa", k_list_pull<true, false, false>, a, pull_pf_);
        else if (cs_nt_)
          launch("list_pull_soa", k_list_pull<true, true, true>, a, pull_pf_);
        else
          launch("list_pull_soa", k_list_pull<true, true, false>, a, pull_pf_);
      } else {
        last ? launch("list_pull_stream_aos", k_list_pull<false, false, false>, a, pull_pf_)
             : launch("list_pull_aos", k_list_pull<false, true, false>, a, pull_pf_);
      }
      cur_ ^= 1;
    }
  }

  template <int MODE>
  void canon(uint64_t c0, uint64_t c1, double* stage, uint64_t seed = 0,
             double amp = 0, double* rho = nullptr, double* u = nullptr) {
    if (c1 <= c0) return;
    ListArgs a = base_args();
    const int g = grid_for(c1 - c0, 256);
    const uint32_t* loc = desc_.blk > 0 ? list_of_canon_.get() : nullptr;
    if (desc_.soa)
      k_list_canon<true, MODE><<<g, 256, 0, stream_>>>(a, buf_[cur_].get(), loc, c0, c1,
                                                       stage, seed, amp, rho, u);
    else
      k_list_canon<false, MODE><<<g, 256, 0, stream_>>>(a, buf_[cur_].get(), loc, c0, c1,
                                                        stage, seed, amp, rho, u);
    LBM_CHECK_LAUNCH();
  }

  void gather_canonical(uint64_t c0, uint64_t count, double* out) override {
    canon<0>(c0, std::min(c0 + count, n_fluid_), out);
  }
  void scatter_canonical(uint64_t c0, uint64_t count, const double* in) override {
    canon<1>(c0, std::min(c0 + count, n_fluid_), const_cast<double*>(in));
  }
  void load_perturbed(uint64_t seed, double amp) override {
    canon<2>(0, n_fluid_, nullptr, seed, amp);
  }
  void macro_fields(double* rho, double* u) override {
    canon<3>(0, n_fluid_, nullptr, 0, 0, rho, u);
  }

  double total_mass() override {
    DevBuf<double> tmp(n_fluid_ * kQ);
    ListArgs a = base_args();
    desc_.soa ? k_list_mass_terms<true><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(
                    a, buf_[cur_].get(), tmp.get())
              : k_list_mass_terms<false><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(
                    a, buf_[cur_].get(), tmp.get());
    LBM_CHECK_LAUNCH();
    return device_sum(tmp.get(), tmp.size(), stream_);
  }

  void export_structure(int32_t* nodes, uint32_t* adj, uint64_t* starts,
                        uint64_t* total) override {
    if (nodes)
      LBM_CUDA(cudaMemcpyAsync(nodes, nodes_.get(), nodes_.bytes(),
                               cudaMemcpyDeviceToHost, stream_));
    if (adj) {
      DevBuf<uint32_t> canon(18 * n_fluid_);
      k_adj_canonical<<<grid_for(18 * n_fluid_, 256), 256, 0, stream_>>>(
          adj_.get(), n_fluid_, canon.get());
      LBM_CHECK_LAUNCH();
      LBM_CUDA(cudaMemcpyAsync(adj, canon.get(), canon.bytes(),
                               cudaMemcpyDeviceToHost, stream_));
      LBM_CUDA(cudaStreamSynchronize(stream_));
    }
    if (starts)
      for (int q = 0; q < kQ; ++q) starts[q] = desc_.soa ? starts_[q] : 0;
    if (total) *total = total_slots_;
    LBM_CUDA(cudaStreamSynchronize(stream_));
  }

  // ria_stats / vector_fraction (kernels_list_aa.cpp:95-140) for the ria/pv
  // names; computed from the run starts of the kernel's own structure.
  // Run coding of the scatter table (build_ria, list_lattice.cpp:206-226) and
  // the device tables of the run-coded odd step.
  void build_ria() {
    DevBuf<uint8_t> is_start(n_fluid_);
    ListArgs a = base_args();
    k_ria_starts<<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(
        adj_.get(), n_fluid_, desc_.soa, a, is_start.get());
    LBM_CHECK_LAUNCH();
    DevBuf<uint32_t> incl(n_fluid_);
    {
      cub::TransformInputIterator<uint32_t, IsStart, const uint8_t*> it(is_start.get(), IsStart{});
      size_t tmp = 0;
      LBM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, it, incl.get(),
                                             static_cast<int64_t>(n_fluid_), stream_));
      DevBuf<uint8_t> t(tmp);
      LBM_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, it, incl.get(),
                                             static_cast<int64_t>(n_fluid_), stream_));
    }
    uint32_t R = 0;
    LBM_CUDA(cudaMemcpyAsync(&R, incl.get() + n_fluid_ - 1, 4, cudaMemcpyDeviceToHost, stream_));
    LBM_CUDA(cudaStreamSynchronize(stream_));
    ria_R_ = R;
    DevBuf<uint32_t> run_start(R);
    const uint64_t warps = ceil_div(n_fluid_, 32);
    ria_run0_.alloc(warps);
    ria_mask_.alloc(warps);
    k_ria_tables<<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, stream_>>>(
        is_start.get(), incl.get(), n_fluid_, run_start.get(), ria_run0_.get(), ria_mask_.get());
    LBM_CHECK_LAUNCH();
    ria_pat_.alloc(uint64_t(R) * 18);
    k_ria_patterns<<<grid_for(uint64_t(R) * 18, 256), 256, 0, stream_>>>(
        adj_.get(), run_start.get(), R, a, ria_pat_.get());
    LBM_CHECK_LAUNCH();
    ria_gpat_.alloc(warps * 18);
    k_ria_group_patterns<<<grid_for(warps * 18, 256), 256, 0, stream_>>>(
        ria_pat_.get(), ria_run0_.get(), ria_mask_.get(), n_fluid_, ria_gpat_.get());
    LBM_CHECK_LAUNCH();
    // run lengths -> vectorizable fraction (list_lattice.cpp:228-236)
    std::vector<uint32_t> h(R);
    LBM_CUDA(cudaMemcpyAsync(h.data(), run_start.get(), uint64_t(R) * 4,
                             cudaMemcpyDeviceToHost, stream_));
    LBM_CUDA(cudaStreamSynchronize(stream_));
    const uint64_t W = static_cast<uint64_t>(desc_.vector_width);
    uint64_t covered = 0;
    for (uint32_t r = 0; r < R; ++r) {
      const uint64_t end = r + 1 < R ? h[r + 1] : n_fluid_;
      covered += (end - h[r]) / W * W;
    }
    ria_runs_ = R;
    ria_vfrac_ = static_cast<double>(covered) / static_cast<double>(n_fluid_);
  }

  bool ria_stats(int64_t* runs, double* vfrac) override {
    if (!desc_.ria) return false;
    *runs = ria_runs_;
    *vfrac = ria_vfrac_;
    return true;
  }

 private:
  int nx_ = 0, ny_ = 0, nz_ = 0;
  std::array<bool, 3> per_{};
  uint64_t starts_[kQ] = {};
  uint64_t total_slots_ = 0;
  bool scatter_ = false;
  bool cs_nt_ = false;
  // index-prefetching persistent odd kernel: measured 4-8 % slower than the
  // one-node-per-thread kernel on B200 (cfg 2/4), kept opt-in
  bool odd_pipe_ = false;
  int sm_count_ = 148;
  int cur_ = 0;
  DevBuf<int32_t> nodes_;
  DevBuf<uint32_t> adj_;
  DevBuf<uint32_t> list_of_canon_;
  DevBuf<double> buf_[2];
  int64_t ria_runs_ = -1;
  double ria_vfrac_ = 0.0;
  uint64_t ria_R_ = 0;
  DevBuf<int32_t> ria_pat_;     // [run][18] relative offsets
  DevBuf<uint32_t> ria_run0_;   // run id of node 32w
  DevBuf<uint32_t> ria_mask_;   // run starts within nodes 32w .. 32w+31
  DevBuf<int32_t> ria_gpat_;    // [group][18] inline pattern or kMixedGroup
  int ria_mode_ = 0;            // 0: run table, 1: group patterns (LBMGPU_RIA_MODE)
  uint64_t pf_ = 0;             // adjacency L2 prefetch distance in nodes (AA odd)
  uint64_t pull_pf_ = 0;        // same for the one-step pull sweeps
};

}  // namespace

std::unique_ptr<Engine> make_list_engine(const Descriptor& d,
                                         const GeomSpec& g,
                                         const Padding& pad) {
  return std::make_unique<ListEngine>(d, g, pad);
}

}  // namespace lbmgpu

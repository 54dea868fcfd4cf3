// List AA run coding (RIA): run tables, patterns, pattern ids and the run-coded odd steps.
// (part of the list-addressing translation unit, included by list.cu)
#pragma once

#include "list_sweeps.cuh"

namespace lbmgpu {

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

// Pattern-id form of the run coding, for lattices whose runs share few
// distinct patterns (a channel: interior, walls, edges): the <= 256 distinct
// rows live in a small table that stays in L1, and every node carries the
// one-byte id of its run's row.  The dependent chain in front of the gathers
// is then one coalesced byte load (prefetched into L2 a wave ahead) and an
// L1 hit, instead of the run-table word and the run's row from L2.
template <typename ID>
__global__ void k_ria_node_ids(const uint32_t* __restrict__ warp_run0,
                               const uint32_t* __restrict__ warp_mask,
                               const ID* __restrict__ run_pid, uint64_t N,
                               ID* __restrict__ nid) {
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < N;
       n += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t lane = static_cast<uint32_t>(n & 31);
    const uint32_t below = (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u)) & ~1u;
    const uint32_t r = warp_run0[n >> 5] + __popc(warp_mask[n >> 5] & below);
    nid[n] = run_pid[r];
  }
}

// ID = uint8_t: <= 256 distinct rows (<= 18 KB, L1-resident; a channel);
// ID = uint16_t / uint32_t: <= 65,536 / 2^20 rows (<= 4.7 / 72 MiB,
// L2-resident; cfg 4 blocks: 144,084 distinct rows of 6,422,500 runs,
// 10 MB) -- the rows then come from L2 instead of the per-run pattern table
// in DRAM (72 B per run, 8.7 nodes per run on cfg 4), for 2-4 B of id per
// node.
// __launch_bounds__(256, 2): <= 128 registers (4 CTAs of 128 threads per
// SM).  Measured alternatives: (128, 5) -- 96 registers, small spill -- 1-2 %
// slower; re-reading the row's offsets after the collision instead of
// keeping them live 3-5 % slower (the loads get hoisted, registers rise).
template <bool CS, typename ID = uint8_t>
__global__ void __launch_bounds__(256, 2)
    k_list_aa_odd_pid(const ListArgs a, const int32_t* __restrict__ ptab,
                      const ID* __restrict__ nid, uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  if (pf && (threadIdx.x & 31) == 0) {  // ids of a later wave -> L2
    const uint64_t m = n + pf;
    if (m < a.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(nid + m));
  }
  const int32_t* p = ptab + uint32_t(__ldg(nid + n)) * 18;
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

// The same pattern-id coding applied to the one-step pull's Gather table
// (experimental, LBMGPU_PULL_PID=1): entry(n, d) = starts[d] + n + row[d-1]
// -- 2-4 B of id per node instead of 72 B of indices; same loads, collision
// and stores as k_list_pull, so bitwise equal.
template <bool COLLIDE, bool CS, typename ID>
__global__ void __launch_bounds__(256, 2)
    k_list_pull_pid(const ListArgs a, const int32_t* __restrict__ ptab,
                    const ID* __restrict__ nid, uint64_t pf) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= a.N) return;
  if (pf && (threadIdx.x & 31) == 0) {
    const uint64_t m = n + pf;
    if (m < a.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(nid + m));
  }
  const int32_t* p = ptab + uint32_t(__ldg(nid + n)) * 18;
  double q[kQ];
  q[0] = a.src[a.starts[0] + n];
#pragma unroll
  for (int d = 1; d < kQ; ++d) q[d] = a.src[int64_t(a.starts[d] + n) + __ldg(p + d - 1)];
  if (COLLIDE) collide(q, a.trt);
  if (!COLLIDE) loads_before_stores();
#pragma unroll
  for (int d = 0; d < kQ; ++d) lst<CS>(a.dst + a.starts[d] + n, q[d]);
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

}  // namespace lbmgpu

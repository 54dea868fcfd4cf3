// Multi-sweep launches for L2-resident lattices (grid barrier; opt-in dataflow).
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include "direct_args.cuh"
#include <cooperative_groups.h>

#include "direct_node.cuh"

namespace lbmgpu {

// ---- fused multi-step sweeps for small lattices ----------------------------
// For lattices that live in L2 (cfg 1: 2 x 40 MB) a sweep takes ~15 us and
// the per-launch fill/drain and launch gaps cost as much as the work.  One
// cooperative launch runs all T sweeps with a grid barrier between them;
// every block walks the nodes grid-stride.  Same per-node bodies, so the
// results are bitwise those of the per-sweep kernels.
struct GridBarrier {
  unsigned* count;
  unsigned* gen;
  int mode;  // 0: counter + generation below, 1: cooperative_groups grid sync
};

__device__ __forceinline__ void grid_sync(const GridBarrier& b) {
  if (b.mode == 1) {
    cooperative_groups::this_grid().sync();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = b.gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(b.count, 1u) == gridDim.x - 1) {
      atomicExch(b.count, 0u);
      __threadfence();
      atomicAdd(b.gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

enum FusedKind { kFusedPush = 0, kFusedPull = 1, kFusedAA = 2 };

template <bool SOA, int KIND, int TPB = 256, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) k_full_fused(DirectArgs a, double* other,
                                                          long steps, GridBarrier bar) {
  const uint32_t G = gridDim.x * blockDim.x;
  auto sweep = [&](auto body) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.count; i += G) {
      const uint32_t n = a.node0 + i;
      Coords c;
      decode_node(a, n, c);
      body(c, n);
    }
  };
  if (KIND == kFusedAA) {
    for (long s = 0; s < steps; s += 2) {
      sweep([&](const Coords& c, uint32_t n) { aa_even_node<SOA, false, true>(a, c, n); });
      grid_sync(bar);
      sweep([&](const Coords& c, uint32_t n) { aa_odd_node<SOA, false, true>(a, c, n); });
      grid_sync(bar);
    }
    return;
  }
  // two grids: a.src -> a.dst, then swap (the host tracks the parity)
  double* bufs[2] = {const_cast<double*>(a.src), other};
  int cur = 0;
  if (KIND == kFusedPull) {
    a.dst = bufs[0];
    sweep([&](const Coords& c, uint32_t n) { collide_node_pass<SOA, true>(a, c, n); });
    grid_sync(bar);
  }
  for (long s = 0; s < steps; ++s) {
    a.src = bufs[cur];
    a.dst = bufs[1 - cur];
    if (KIND == kFusedPush)
      sweep([&](const Coords& c, uint32_t n) { push_node<SOA, false, true>(a, c, n); });
    else if (s + 1 < steps)
      sweep([&](const Coords& c, uint32_t n) { pull_node<SOA, true, false, true>(a, c, n); });
    else
      sweep([&](const Coords& c, uint32_t n) { pull_node<SOA, false, false, true>(a, c, n); });
    grid_sync(bar);
    cur ^= 1;
  }
}

// ---- the same multi-sweep run as a plane-level dataflow --------------------
// No grid barrier: the T sweeps are cut into tasks (sweep s, plane z, chunk i)
// of blockDim nodes.  A task of sweep s > 0 waits until sweep s-1 has
// finished planes z-1, z, z+1 (z wrapped); that covers every read and write
// hazard of push, pull and AA (each sweep touches only the planes next to its
// own, and the chains close transitively -- DESIGN.md section 4).
// plane_done[z] counts finished chunks of plane z over all sweeps, so "sweep
// s-1 done on z" is plane_done[z] >= s * chunks_per_plane (release add by the
// finishing block, acquire load by the waiting one; lattice loads are
// ld.global.cg, so no stale L1 line is read).  All blocks are co-resident
// (cooperative launch).  Blocks that finish their part of a sweep start the
// next one instead of idling at a barrier.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool SOA, int KIND, int TPB = 256, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) k_full_flow(DirectArgs a, double* other, long sweeps,
                                                   unsigned* plane_done, unsigned base) {
  // Tasks are blockDim-node chunks run by whole blocks.  (32-node warp
  // tasks without block barriers measured 2x slower: the release/acquire
  // fences per task dominate.)
  const uint32_t lane = threadIdx.x;
  const uint64_t worker = blockIdx.x;
  const uint64_t workers = gridDim.x;
  const uint32_t cpp = (a.P + blockDim.x - 1) / blockDim.x;  // chunks per plane
  const uint64_t per_sweep = uint64_t(a.nzl) * cpp;
  const uint64_t total = per_sweep * uint64_t(sweeps);
  double* bufs[2] = {const_cast<double*>(a.src), other};
  // Static round-robin assignment (block b: tasks b, b + grid, ...): every
  // block runs its tasks in increasing order, so the smallest unfinished task
  // is always running and its dependencies (all smaller) are done.  Sweep s
  // visits the planes starting at plane 2s: sweep s's i-th plane then needs
  // sweep s-1's (i+1)..(i+3)-th planes, dispatched about a whole sweep
  // earlier -- without the rotation the z wrap would make the first plane of
  // every sweep wait for the last plane of the previous one.
  auto where = [&](uint64_t task, uint32_t& s, uint32_t& z, uint32_t& chunk) {
    s = static_cast<uint32_t>(task / per_sweep);
    const uint32_t rem = static_cast<uint32_t>(task - uint64_t(s) * per_sweep);
    const uint32_t zi = rem / cpp;
    chunk = rem - zi * cpp;
    z = static_cast<uint32_t>((zi + 2ull * s) % a.nzl);
  };
  // lanes 0-2 watch planes z-1, z, z+1 of the previous sweep
  auto watched = [&](uint32_t z) {
    return lane == 0 ? (z == 0 ? a.nzl - 1 : z - 1)
         : lane == 1 ? z
                     : (z + 1 == a.nzl ? 0 : z + 1);
  };
  // The counters a task needs are read one task ahead (relaxed; re-polled
  // only if not yet enough); the acquire is a fence after the observing
  // read, so in the common case (dependencies finished about a sweep ago)
  // the check puts no L2 round trip on the critical path.
  unsigned seen = 0;
  if (lane < 3 && worker < total) {
    uint32_t s, z, chunk;
    where(worker, s, z, chunk);
    seen = ld_relaxed(plane_done + watched(z));
  }
  for (uint64_t task = worker; task < total; task += workers) {
    uint32_t s, z, chunk;
    where(task, s, z, chunk);
    if (s > 0) {
      if (lane < 3) {
        const unsigned need = base + s * cpp;  // wrap-safe comparisons
        while (static_cast<int>(seen - need) < 0) {
          __nanosleep(32);
          seen = ld_relaxed(plane_done + watched(z));
        }
        __threadfence();
      }
      __syncthreads();
    }
    if (lane < 3 && task + workers < total) {
      uint32_t s2, z2, c2;
      where(task + workers, s2, z2, c2);
      seen = ld_relaxed(plane_done + watched(z2));
    }
    const uint32_t x = chunk * blockDim.x + lane;
    if (x < a.P) {
      const uint32_t n = z * a.P + x;
      Coords c;
      decode_node(a, n, c);
      if (KIND == kFusedAA) {
        if (s & 1)
          aa_odd_node<SOA, false, true>(a, c, n);
        else
          aa_even_node<SOA, false, true>(a, c, n);
      } else if (KIND == kFusedPush) {
        a.src = bufs[s & 1];
        a.dst = bufs[(s & 1) ^ 1];
        push_node<SOA, false, true>(a, c, n);
      } else if (s == 0) {  // pull: collide pass on the current grid
        a.dst = bufs[0];
        collide_node_pass<SOA, true>(a, c, n);
      } else {
        a.src = bufs[(s - 1) & 1];
        a.dst = bufs[s & 1];
        if (s + 1 < sweeps)
          pull_node<SOA, true, false, true>(a, c, n);
        else
          pull_node<SOA, false, false, true>(a, c, n);
      }
    }
    __syncthreads();  // orders the block's stores before thread 0's release
    if (lane == 0) red_release_add(plane_done + z, 1u);
  }
}

}  // namespace lbmgpu

// Multi-sweep launches for L2-resident lattices (cooperative grid barrier).
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
__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }

enum FusedKind { kFusedPush = 0, kFusedPull = 1, kFusedAA = 2 };

template <bool SOA, int KIND, int TPB = 256, int MINB = 1>
__global__ void __launch_bounds__(TPB, MINB) k_full_fused(DirectArgs a, double* other,
                                                          long steps) {
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
      grid_sync();
      sweep([&](const Coords& c, uint32_t n) { aa_odd_node<SOA, false, true>(a, c, n); });
      grid_sync();
    }
    return;
  }
  // two grids: a.src -> a.dst, then swap (the host tracks the parity)
  double* bufs[2] = {const_cast<double*>(a.src), other};
  int cur = 0;
  if (KIND == kFusedPull) {
    a.dst = bufs[0];
    sweep([&](const Coords& c, uint32_t n) { collide_node_pass<SOA, true>(a, c, n); });
    grid_sync();
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
    grid_sync();
    cur ^= 1;
  }
}

}  // namespace lbmgpu

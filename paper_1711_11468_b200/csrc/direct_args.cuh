// Kernel arguments of the direct-addressing sweeps (direct.cu and its .cuh parts).
#pragma once

#include "lbm.hpp"

namespace lbmgpu {

struct DirectArgs {
  const double* src;
  double* dst;
  const uint8_t* flags;  // own planes, (z*ny + y)*nx + x, 1 = solid
  const uint32_t* tmask; // push only (may be null): bit d = target x + c_d solid
  uint32_t nx, ny, nzl;  // own extents
  uint32_t zoff;         // storage plane of own plane 0
  uint32_t zwrap;        // 1: single part, wrap z over own planes
  uint32_t P;            // nx*ny
  FastDiv fdx, fdP;      // n / nx, n / P
  uint32_t node0, count; // own-node range of this launch
  TrtArgs trt;
  // Analytic solid test for the built-in geometries (geometry.cpp:48-104),
  // so the AA sweeps need no flag load before their PDF loads; kind 4
  // (custom FlagField) reads `flags`.
  int geom;              // 0 channel, 1 slit, 2 pipe, 3 blocks, 4 custom
  int gny, gnz, z0;      // global ny, nz and the slab's first global z
  int period, spacing;   // blocks
  long long d2;          // pipe: D^2
  // AA odd step, interior nodes (no x/y/z wrap): element offset of
  // direction d's gather/scatter slot, (x - c_d, opp d), from the node's own
  // slot-0 element.  One 64-bit add per direction instead of the wrapped
  // coordinate arithmetic; layout-specific, filled on the host.
  long long odd_off[kQ];
  // AoS gather/scatter sweeps: traverse rows in y-bands of `band` rows, z
  // before y inside a band, so the z +- 1 rows whose records a row's
  // gathers touch are processed close in time (L2 reuse); 0 = plain order.
  uint32_t band;
};

// Solid flag of own node (x, y, own-plane z) without touching memory for the
// built-in kinds; the integer tests are the reference's.
__device__ __forceinline__ bool solid_node(const DirectArgs& a, uint32_t x, uint32_t y,
                                           uint32_t z, uint32_t n) {
  const int zg = static_cast<int>(z) + a.z0;
  const int yy = static_cast<int>(y);
  switch (a.geom) {
    case 0:
      return yy == 0 || yy == a.gny - 1 || zg == 0 || zg == a.gnz - 1;
    case 1:
      return zg == 0 || zg == a.gnz - 1;
    case 2: {
      const long long dy = 2LL * yy - (a.gny - 1), dz = 2LL * zg - (a.gnz - 1);
      return dy * dy + dz * dz > a.d2;
    }
    case 3:
      return static_cast<int>(x) % a.period >= a.spacing && yy % a.period >= a.spacing &&
             zg % a.period >= a.spacing;
    default:
      return a.flags[n] != 0;
  }
}

}  // namespace lbmgpu

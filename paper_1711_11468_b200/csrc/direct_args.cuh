// Kernel arguments of the direct-addressing sweeps (direct.cu, direct_tma.cu).
#pragma once

#include "lbm.hpp"

namespace lbmgpu {

struct DirectArgs {
  const double* src;
  double* dst;
  const uint8_t* flags;  // own planes, (z*ny + y)*nx + x, 1 = solid
  uint32_t nx, ny, nzl;  // own extents
  uint32_t zoff;         // storage plane of own plane 0
  uint32_t zwrap;        // 1: single part, wrap z over own planes
  uint32_t P;            // nx*ny
  FastDiv fdx, fdP;      // n / nx, n / P
  uint32_t node0, count; // own-node range of this launch
  TrtArgs trt;
};

constexpr uint32_t kTmaTile = 256;  // nodes per TMA row tile

// TMA-staged AA sub-step (direct_tma.cu); false = shape not supported.
bool launch_aa_tma(bool odd, const DirectArgs& a, int sm_count, int stages,
                   cudaStream_t s);

}  // namespace lbmgpu

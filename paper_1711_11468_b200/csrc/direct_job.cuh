// Pipelined job of the direct AA lattices (DirectEngine::run_job, direct.cu):
// the z-chunk <-> staging transfer kernel and the column census it needs.
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include "direct_args.cuh"

namespace lbmgpu {

// Column census: for every (x, y) column of the box, the number of fluid
// planes and the first / last fluid plane (flags: (z*ny + y)*nx + x, 1 =
// solid).  One thread per column, plane loop (coalesced across columns).
__global__ void k_job_columns(const uint8_t* __restrict__ flags, uint64_t P, uint32_t nz,
                              uint32_t* __restrict__ census /* [P][3]: count, zmin, zmax */) {
  for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < P;
       c += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t cnt = 0, zmin = 0xffffffffu, zmax = 0;
    for (uint32_t z = 0; z < nz; ++z)
      if (!flags[uint64_t(z) * P + c]) {
        ++cnt;
        zmin = min(zmin, z);
        zmax = z;
      }
    census[3 * c] = cnt;
    census[3 * c + 1] = zmin;
    census[3 * c + 2] = zmax;
  }
}

// Planes [z0, z0 + w) of every fluid column <-> staging [R][w][19]: column r
// (the r-th non-empty column in the reference's x-major order) holds
// canonical rows r*w .. r*w + w-1 of the chunk, i.e. the host's canonical
// rows r*nzf + (z - za) -- a 2-D copy.  A CTA moves the tile of kJobTx
// consecutive x of one y row through shared memory: the lattice side as
// 256-byte x rows per (plane, slot), the staging side as one contiguous
// w*19-double block per column (col_of: in-plane offset -> column, ~0 =
// no fluid), so both sides are coalesced.
constexpr int kJobTx = 32;
template <bool SOA, bool TO_STAGING>
__global__ void __launch_bounds__(256) k_job_chunk(double* __restrict__ buf,
                                                   const uint32_t* __restrict__ col_of,
                                                   uint32_t w, uint32_t z0, uint32_t nx,
                                                   uint32_t ny, double* __restrict__ staging) {
  extern __shared__ double jt[];  // [kJobTx][w*19 + 1] (odd stride: no bank conflicts)
  __shared__ int slot_of[kQ];
  const uint64_t P = uint64_t(nx) * ny;
  const uint32_t tiles_x = (nx + kJobTx - 1) / kJobTx;
  const uint32_t y = blockIdx.x / tiles_x, x0 = (blockIdx.x % tiles_x) * kJobTx;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  const uint32_t W = w * kQ;  // doubles per column block
  const uint32_t Ws = W + 1;  // its shared-memory stride
  if (t < uint32_t(kQ)) slot_of[t] = dslot(static_cast<int>(t));
  auto lattice = [&](uint32_t x, uint32_t i, int slot) -> uint64_t {
    const uint64_t z = z0 + i;
    return SOA ? (z * kQ + slot) * P + uint64_t(y) * nx + x
               : (z * P + uint64_t(y) * nx + x) * kQ + slot;
  };
  if (!TO_STAGING) {  // staging blocks -> shared (one warp per column)
    for (uint32_t c = warp; c < kJobTx; c += nwarps) {
      const uint32_t x = x0 + c;
      if (x >= nx) continue;
      const uint32_t r = col_of[uint64_t(y) * nx + x];
      if (r == 0xffffffffu) continue;
      const double* src = staging + uint64_t(r) * W;
      for (uint32_t e = lane; e < W; e += 32) jt[c * Ws + e] = src[e];
    }
  }
  __syncthreads();
  // lattice side: warp = one (plane, slot) x row at a time
  {
    const uint32_t x = x0 + lane;
    const bool fluid_col = x < nx && col_of[uint64_t(y) * nx + x] != 0xffffffffu;
    for (uint32_t k = warp; k < w * kQ; k += nwarps) {
      const uint32_t i = k / kQ;
      const int d = static_cast<int>(k - i * kQ);
      if (!fluid_col) continue;
      double* p = buf + lattice(x, i, slot_of[d]);
      double* s = jt + lane * Ws + i * kQ + d;
      if (TO_STAGING)
        *s = *p;
      else
        *p = *s;
    }
  }
  if (TO_STAGING) {  // shared -> staging blocks
    __syncthreads();
    for (uint32_t c = warp; c < kJobTx; c += nwarps) {
      const uint32_t x = x0 + c;
      if (x >= nx) continue;
      const uint32_t r = col_of[uint64_t(y) * nx + x];
      if (r == 0xffffffffu) continue;
      double* dst = staging + uint64_t(r) * W;
      for (uint32_t e = lane; e < W; e += 32) dst[e] = jt[c * Ws + e];
    }
  }
}

}  // namespace lbmgpu

// Direct AoS sweeps through shared-memory tiles (TMA bulk copies).
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include "direct_args.cuh"
#include "direct_node.cuh"
#include "tma.cuh"

namespace lbmgpu {

// AoS own-record sweeps (AA even: own slots -> opposite slots; the pull's
// collide pass: in place) on a tile of kAosTile consecutive nodes staged
// through shared memory.  A thread's record lives at sh[t*19 .. t*19+18] and
// only that thread touches it between the barriers; solid records are
// written back unchanged.  Same per-node arithmetic as aa_even_node /
// collide_node_pass.
constexpr int kAosTile = 128;
template <bool EVEN>
__global__ void __launch_bounds__(kAosTile) k_full_aos_tile(const DirectArgs a) {
  __shared__ __align__(128) double sh[kAosTile * kQ];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t n0 = a.node0 + blockIdx.x * kAosTile;
  const uint32_t cnt = min(uint32_t(kAosTile), a.node0 + a.count - n0);
  // record of own node n: storage plane z + zoff, i.e. n + zoff * P
  double* g = a.dst + (uint64_t(n0) + uint64_t(a.zoff) * a.P) * kQ;
  aos_tile_load<kAosTile>(sh, g, cnt, &bar);
  if (threadIdx.x < cnt) {
    const uint32_t n = n0 + threadIdx.x;
    Coords c;
    decode_node(a, n, c);
    if (!solid_node(a, c.x, c.y, c.z, n)) {
      double* r = sh + threadIdx.x * kQ;
      double q[kQ];
#pragma unroll
      for (int d = 0; d < kQ; ++d) q[d] = r[dslot(d)];
      collide(q, a.trt);
#pragma unroll
      for (int d = 0; d < kQ; ++d) r[dslot(EVEN ? opp(d) : d)] = q[d];
    }
  }
  aos_tile_store<kAosTile>(g, sh, cnt);
}

// AoS pull through 3-D halo tiles.  A block owns a 16 x 4 x 4 (x, y, z) tile
// of nodes; the 6 x 6 source rows around it, each as 20 whole records
// (x0-2 .. x0+17, i.e. 16-byte aligned), arrive by 1-D TMA bulk copies into
// shared memory (rows wrapped on y and z, row segments split at the periodic
// x wrap), every node gathers its 19 values there, and the tile's own
// destination records leave by 16 bulk stores after the block barrier.  Each
// source record is fetched by the ~2.25 tiles around it instead of as 19
// separate 32-byte sectors; destination records are written whole.  Needs a
// single part with nx % 16 == 0, ny % 4 == 0, nz % 4 == 0.
constexpr int kPtX = 16;
constexpr int kPtW = kPtX + 4;                           // records per halo row
constexpr uint32_t kPtRowBytes = kPtW * kQ * 8;         // 3040
template <int kPtY, int kPtZ>
constexpr size_t pt_smem() {
  return size_t((kPtY + 2) * (kPtZ + 2)) * kPtRowBytes + 16;
}
// Halo rows of a 16 x TY x TZ tile at (x0, y0, z0) from AoS grid `src` into
// shared memory `sh` (block-wide; ends with the copies in flight on `bar`).
template <int kPtY, int kPtZ>
__device__ __forceinline__ void pt_load_halo(const DirectArgs& a, const double* src, double* sh,
                                             uint64_t* bar, uint32_t x0, uint32_t y0,
                                             uint32_t z0) {
  constexpr int kPtRows = (kPtY + 2) * (kPtZ + 2);
  const uint64_t nx = a.nx;
  auto rec = [&](uint32_t zs, uint32_t y, uint32_t x) {  // record pointer (AoS)
    return src + ((uint64_t(zs) * a.ny + y) * nx + x) * kQ;
  };
  const uint32_t t = threadIdx.x;
  if (t == 0) {
    tma::mbar_init(bar, 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  // warp 0 issues the row copies: lane l handles halo rows l and l + 32
  if (t < 32) {
    if (t == 0) tma::mbar_arrive_expect_tx(bar, kPtRows * kPtRowBytes);
    __syncwarp();
    for (uint32_t row = t; row < uint32_t(kPtRows); row += 32) {
      const uint32_t hy = row % (kPtY + 2), hz = row / (kPtY + 2);
      const uint32_t y = (y0 + a.ny + hy - 1) % a.ny;
      const uint32_t z = (z0 + a.nzl + hz - 1) % a.nzl;  // single part: zwrap
      double* dst = sh + size_t(row) * kPtW * kQ;
      if (x0 >= 2 && x0 + kPtX + 2 <= nx) {
        tma::bulk_g2s(dst, rec(z, y, x0 - 2), kPtRowBytes, bar);
      } else {  // split at the x wrap: pieces of records [x0-2, x0+18) mod nx
        uint32_t h = 0;
        while (h < uint32_t(kPtW)) {
          const uint32_t x = uint32_t((int64_t(x0) - 2 + h + nx) % nx);
          const uint32_t len = min(uint32_t(kPtW) - h, uint32_t(nx - x));
          tma::bulk_g2s(dst + size_t(h) * kQ, rec(z, y, x), len * kQ * 8, bar);
          h += len;
        }
      }
    }
  }
}

template <bool COLLIDE, int kPtY, int kPtZ>
__global__ void __launch_bounds__(kPtX * kPtY * kPtZ) k_full_pull_aos_tile3d(const DirectArgs a) {
  constexpr int kPtRows = (kPtY + 2) * (kPtZ + 2);  // halo rows
  extern __shared__ __align__(128) unsigned char pt_smem[];
  double* sh = reinterpret_cast<double*>(pt_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(pt_smem + size_t(kPtRows) * kPtRowBytes);
  const uint32_t tilesx = a.nx / kPtX, tilesy = a.ny / kPtY;
  const uint32_t b = blockIdx.x;
  const uint32_t x0 = (b % tilesx) * kPtX;
  const uint32_t y0 = ((b / tilesx) % tilesy) * kPtY;
  const uint32_t z0 = (b / (tilesx * tilesy)) * kPtZ;
  const uint64_t nx = a.nx;
  const uint32_t t = threadIdx.x;
  pt_load_halo<kPtY, kPtZ>(a, a.src, sh, bar, x0, y0, z0);
  const uint32_t tx = t % kPtX, ty = (t / kPtX) % kPtY, tz = t / (kPtX * kPtY);
  const uint32_t n = ((z0 + tz) * a.ny + (y0 + ty)) * a.nx + (x0 + tx);
  const bool solid = solid_node(a, x0 + tx, y0 + ty, z0 + tz, n);
  tma::mbar_wait(bar, 0);
  auto at = [&](int hx, int hy, int hz) {
    return sh + (size_t(hz * (kPtY + 2) + hy) * kPtW + hx) * kQ;
  };
  double q[kQ];
  q[0] = at(tx + 2, ty + 1, tz + 1)[dslot(0)];
#pragma unroll
  for (int d = 1; d < kQ; ++d)
    q[d] = at(int(tx) + 2 - cx(d), int(ty) + 1 - cy(d), int(tz) + 1 - cz(d))[dslot(d)];
  if (COLLIDE && !solid) collide(q, a.trt);
  __syncthreads();  // every gather done: the centre records may be overwritten
  double* own = at(tx + 2, ty + 1, tz + 1);
  own[dslot(0)] = q[0];
#pragma unroll
  for (int d = 1; d < kQ; ++d) own[solid ? dslot(opp(d)) : dslot(d)] = q[d];
  tma::fence_proxy_async();
  __syncthreads();
  if (t < uint32_t(kPtY * kPtZ)) {  // one bulk store per centre row
    const uint32_t ry = t % kPtY, rz = t / kPtY;
    double* g = a.dst + ((uint64_t(z0 + rz) * a.ny + (y0 + ry)) * nx + x0) * kQ;
    tma::bulk_s2g(g, at(2, ry + 1, rz + 1), kPtX * kQ * 8);
    tma::bulk_commit();
    tma::bulk_wait_read0();
  }
}

// AoS AA odd step with the gathers through the same 3-D halo tiles: the
// tile's source rows arrive by TMA as whole records, each node reads its 18
// neighbour values (x - c_d, opp d) in shared memory, and writes them back to
// global memory slot by slot (every slot is read and written by exactly one
// node in this sub-step, so the other, possibly stale, slots of the staged
// records are never used).
template <int kPtY, int kPtZ>
__global__ void __launch_bounds__(kPtX * kPtY * kPtZ) k_full_aa_odd_aos_tile3d(const DirectArgs a) {
  constexpr int kPtRows = (kPtY + 2) * (kPtZ + 2);
  extern __shared__ __align__(128) unsigned char pt_smem[];
  double* sh = reinterpret_cast<double*>(pt_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(pt_smem + size_t(kPtRows) * kPtRowBytes);
  const uint32_t tilesx = a.nx / kPtX, tilesy = a.ny / kPtY;
  const uint32_t b = blockIdx.x;
  const uint32_t x0 = (b % tilesx) * kPtX;
  const uint32_t y0 = ((b / tilesx) % tilesy) * kPtY;
  const uint32_t z0 = (b / (tilesx * tilesy)) * kPtZ;
  const uint32_t t = threadIdx.x;
  pt_load_halo<kPtY, kPtZ>(a, a.dst, sh, bar, x0, y0, z0);
  const uint32_t tx = t % kPtX, ty = (t / kPtX) % kPtY, tz = t / (kPtX * kPtY);
  const uint32_t n = ((z0 + tz) * a.ny + (y0 + ty)) * a.nx + (x0 + tx);
  Coords c;
  decode_node(a, n, c);
  const bool solid = solid_node(a, c.x, c.y, c.z, n);
  tma::mbar_wait(bar, 0);
  if (solid) return;
  auto at = [&](int hx, int hy, int hz) {
    return sh + (size_t(hz * (kPtY + 2) + hy) * kPtW + hx) * kQ;
  };
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d)
    q[d] = at(int(tx) + 2 - cx(d), int(ty) + 1 - cy(d), int(tz) + 1 - cz(d))[dslot(opp(d))];
  collide(q, a.trt);
  const Idx<false> I{a.P, a.nx, a.ny};
#pragma unroll
  for (int d = 0; d < kQ; ++d)
    a.dst[I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)])] = q[opp(d)];
}

}  // namespace lbmgpu

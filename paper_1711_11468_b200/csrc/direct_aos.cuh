// Direct AoS sweeps through shared-memory tiles (TMA bulk copies).
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include <type_traits>

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
// staged rows of a 16 x TY x TZ tile: the (TY+2) x (TZ+2) halo rows, or
// (HALO = false) only the TY x TZ own rows
template <int kPtY, int kPtZ, bool HALO = true>
__host__ __device__ constexpr int pt_rows() {
  return HALO ? (kPtY + 2) * (kPtZ + 2) : kPtY * kPtZ;
}
template <int kPtY, int kPtZ, bool HALO = true>
constexpr size_t pt_smem() {
  return size_t(pt_rows<kPtY, kPtZ, HALO>()) * kPtRowBytes + 16;
}
// Rows of a 16 x TY x TZ tile at (x0, y0, z0) from AoS grid `src` into
// shared memory `sh`, each as 20 whole records x0-2 .. x0+17 (block-wide;
// ends with the copies in flight on `bar`): the halo rows, staged row
// hz * (TY+2) + hy for halo position (hy, hz), or (HALO = false) the own
// rows, staged row (hz-1) * TY + (hy-1).
template <int kPtY, int kPtZ, bool HALO = true>
__device__ __forceinline__ void pt_load_halo(const DirectArgs& a, const double* src, double* sh,
                                             uint64_t* bar, uint32_t x0, uint32_t y0,
                                             uint32_t z0) {
  constexpr int kPtRows = pt_rows<kPtY, kPtZ, HALO>();
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
      const uint32_t hy = HALO ? row % (kPtY + 2) : row % kPtY + 1;
      const uint32_t hz = HALO ? row / (kPtY + 2) : row / kPtY + 1;
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

// Tile of this CTA.  The grid is 3-D so that no division is needed and the
// launch order (x fastest, then y, then z) is the traversal order: plain
// (a.band <= 1): grid (nx/16, ny/TY, nz/TZ); banded (a.band = by, a power of
// two dividing ny/TY): grid (nx/16, by * nz/TZ, ny/TY/by) -- the (y, z)
// tiles in blocks of by y tiles, y fastest inside a block, then z, then the
// next block.  Blocking keeps a tile's z neighbours by * (nx / 16) launch
// positions away, so the records both touch are still in L2.  tile_grid
// (direct.cu) builds the grid.
template <int kPtY, int kPtZ>
__device__ __forceinline__ void tile_origin(const DirectArgs& a, uint32_t& x0, uint32_t& y0,
                                            uint32_t& z0) {
  x0 = blockIdx.x * kPtX;
  if (a.band > 1) {
    const uint32_t by = a.band, w = blockIdx.y;
    y0 = (blockIdx.z * by + (w & (by - 1))) * kPtY;
    z0 = (w >> (31 - __clz(by))) * kPtZ;
  } else {
    y0 = blockIdx.y * kPtY;
    z0 = blockIdx.z * kPtZ;
  }
}

// No node of the tile at (x0, y0, z0) has a wrapped neighbour: every
// neighbour record sits at a fixed element offset from the node's own record
// (CTA-uniform, so the gathers / scatters outside the staged rows need no
// coordinate arithmetic).
template <int kPtY, int kPtZ>
__device__ __forceinline__ bool tile_inner(const DirectArgs& a, uint32_t x0, uint32_t y0,
                                           uint32_t z0) {
  return x0 >= 1 && x0 + kPtX < a.nx && y0 >= 1 && y0 + kPtY < a.ny && z0 >= 1 &&
         z0 + kPtZ < a.nzl && a.zoff == 0;
}

// HALO = false (the default, measured faster): only the tile's own source
// rows are staged, as in the AA odd step below; the face nodes' gathers
// from y / z halo rows are loaded from global memory ahead of the copies.
template <bool COLLIDE, int kPtY, int kPtZ, bool HALO = false>
__global__ void __launch_bounds__(kPtX * kPtY * kPtZ, HALO ? 1 : 3)
    k_full_pull_aos_tile3d(const DirectArgs a) {
  constexpr int kPtRows = pt_rows<kPtY, kPtZ, HALO>();
  extern __shared__ __align__(128) unsigned char pt_smem[];
  double* sh = reinterpret_cast<double*>(pt_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(pt_smem + size_t(kPtRows) * kPtRowBytes);
  uint32_t x0, y0, z0;
  tile_origin<kPtY, kPtZ>(a, x0, y0, z0);
  const uint64_t nx = a.nx;
  const uint32_t t = threadIdx.x;
  pt_load_halo<kPtY, kPtZ, HALO>(a, a.src, sh, bar, x0, y0, z0);
  const uint32_t tx = t % kPtX, ty = (t / kPtX) % kPtY, tz = t / (kPtX * kPtY);
  const uint32_t n = ((z0 + tz) * a.ny + (y0 + ty)) * a.nx + (x0 + tx);
  const bool solid = solid_node(a, x0 + tx, y0 + ty, z0 + tz, n);
  auto at = [&](int hx, int hy, int hz) {
    const int row = HALO ? hz * (kPtY + 2) + hy : (hz - 1) * kPtY + (hy - 1);
    return sh + (size_t(row) * kPtW + hx) * kQ;
  };
  auto staged = [](int hy, int hz) { return HALO || (hy >= 1 && hy <= kPtY && hz >= 1 && hz <= kPtZ); };
  double q[kQ];
  if (!HALO) {  // gathers from rows that are not staged: now, ahead of the copies
    if (tile_inner<kPtY, kPtZ>(a, x0, y0, z0)) {
      // record of x - c_d: a fixed offset from the own record (odd_off is the
      // AA form, slot opp(d); the pull reads slot d of the same record)
      const double* own = a.src + uint64_t(n) * kQ;
#pragma unroll
      for (int d = 1; d < kQ; ++d) {
        const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
        if (!staged(hy, hz)) q[d] = own[a.odd_off[d] + (dslot(d) - dslot(opp(d)))];
      }
    } else {
      const Idx<false> I{a.P, a.nx, a.ny};
      Coords c;
      fill_coords(a, x0 + tx, y0 + ty, z0 + tz, c);
#pragma unroll
      for (int d = 1; d < kQ; ++d) {
        const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
        if (!staged(hy, hz))
          q[d] = a.src[I(c.Z[1 - cz(d)], dslot(d), c.Y[1 - cy(d)], c.X[1 - cx(d)])];
      }
    }
  }
  tma::mbar_wait(bar, 0);
  q[0] = at(tx + 2, ty + 1, tz + 1)[dslot(0)];
#pragma unroll
  for (int d = 1; d < kQ; ++d) {
    const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
    if (staged(hy, hz)) q[d] = at(int(tx) + 2 - cx(d), hy, hz)[dslot(d)];
  }
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

// c_x + 1 (resp. c_y + 1, c_z + 1) of the direction stored in slot s, as
// 2-bit fields of one constant: a register shift per element instead of a
// table lookup with a lane-dependent index.
template <int AXIS>
__host__ __device__ constexpr uint64_t slot_c_bits() {
  uint64_t m = 0;
  for (int s = 0; s < kQ; ++s) {
    const int d = ddir(s);
    const int c = AXIS == 0 ? cx(d) : AXIS == 1 ? cy(d) : cz(d);
    m |= uint64_t(c + 1) << (2 * s);
  }
  return m;
}

// Which elements of a staged row (20 records x 19 slots, element i = lane +
// 32 j) a tile owns, per lane: bit j of mx = the slot's owner (record x - c_x
// of the slot's direction) lies inside the tile in x; of ypos / yneg / zpos /
// zneg = the slot's direction has c_y (c_z) = +1 / -1.  Constant per lane,
// so built at compile time and read as five coalesced words.
constexpr int kOwnRowElems = kPtW * kQ;           // 380 doubles per staged row
constexpr int kOwnJ = (kOwnRowElems + 31) / 32;  // elements per lane
struct OwnMasks {
  uint32_t mx[32], ypos[32], yneg[32], zpos[32], zneg[32];
};
constexpr OwnMasks make_own_masks() {
  OwnMasks m{};
  constexpr uint64_t kX = slot_c_bits<0>(), kY = slot_c_bits<1>(), kZ = slot_c_bits<2>();
  for (int lane = 0; lane < 32; ++lane)
    for (int jj = 0; jj < kOwnJ; ++jj) {
      const int i = lane + 32 * jj;
      if (i >= kOwnRowElems) continue;
      const int hx = i / kQ, s = i - hx * kQ;
      const int ox = hx + 1 - static_cast<int>((kX >> (2 * s)) & 3u);
      const int ey = static_cast<int>((kY >> (2 * s)) & 3u) - 1;
      const int ez = static_cast<int>((kZ >> (2 * s)) & 3u) - 1;
      if (ox >= 2 && ox < 2 + kPtX) m.mx[lane] |= 1u << jj;
      if (ey > 0) m.ypos[lane] |= 1u << jj;
      if (ey < 0) m.yneg[lane] |= 1u << jj;
      if (ez > 0) m.zpos[lane] |= 1u << jj;
      if (ez < 0) m.zneg[lane] |= 1u << jj;
    }
  return m;
}
__device__ const OwnMasks kOwnMasks = make_own_masks();

// AoS AA odd step through the same 3-D halo tiles, both ways.  The tile's
// source rows arrive by TMA as whole records; each node reads its 19 values
// (x - c_d, opp d) in shared memory and collides.  The slot a node gathers
// direction d from is the one it scatters opp(d) to (kernels_full_aa.cpp:
// 83-92), and slot s of record r is read and written in this sub-step only
// by node r - c_s (s = 0: r itself).  Results whose record lies in one of
// the tile's own (y, z) rows go back into the shared-memory copy; those
// rows then leave by coalesced 8-byte stores of exactly the slots whose
// owner lies in the tile (no slot has two writers; solid owners store
// their unchanged value; slots owned by other CTAs are neither used nor
// written).  Results for records in the y / z halo rows -- a minority,
// from the tile's face nodes -- are stored straight to global memory.  The
// own rows thus leave as full 32-byte sectors instead of one sector per
// scattered 8-byte element.
// HALO = false (the default, measured faster): only the tile's own rows are
// staged (48.6 KB, so 3 CTAs/SM at <= 80 registers instead of 2 of 109 KB);
// a node's entries into the y / z halo rows (face nodes only) are loaded
// from global memory ahead of the copies, and their results are stored
// there directly as before.  cfg-5 box: odd step 3,098 -> 3,433 GB/s
// ((256, 2): 120 registers, 3,193; (256, 4): 64 registers + spills, 2,821).
template <int kPtY, int kPtZ, bool HALO = false>
__global__ void __launch_bounds__(kPtX * kPtY * kPtZ, HALO ? 1 : 3)
    k_full_aa_odd_aos_tile3d(const DirectArgs a) {
  constexpr int kPtRows = pt_rows<kPtY, kPtZ, HALO>();
  constexpr int kT = kPtX * kPtY * kPtZ;
  constexpr int kRowElems = kPtW * kQ;  // 380 doubles per staged row
  extern __shared__ __align__(128) unsigned char pt_smem[];
  double* sh = reinterpret_cast<double*>(pt_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(pt_smem + size_t(kPtRows) * kPtRowBytes);
  uint32_t x0, y0, z0;
  tile_origin<kPtY, kPtZ>(a, x0, y0, z0);
  const uint32_t t = threadIdx.x;
  pt_load_halo<kPtY, kPtZ, HALO>(a, a.dst, sh, bar, x0, y0, z0);
  const uint32_t tx = t % kPtX, ty = (t / kPtX) % kPtY, tz = t / (kPtX * kPtY);
  const uint32_t n = ((z0 + tz) * a.ny + (y0 + ty)) * a.nx + (x0 + tx);
  const bool solid = solid_node(a, x0 + tx, y0 + ty, z0 + tz, n);
  auto at = [&](int hx, int hy, int hz) {
    const int row = HALO ? hz * (kPtY + 2) + hy : (hz - 1) * kPtY + (hy - 1);
    return sh + (size_t(row) * kPtW + hx) * kQ;
  };
  auto staged = [](int hy, int hz) { return HALO || (hy >= 1 && hy <= kPtY && hz >= 1 && hz <= kPtZ); };
  // Entry (x - c_d, opp d) of a node outside the staged rows: a fixed offset
  // from the own record when no node of the tile wraps (INNER, CTA-uniform:
  // one instantiation of the body per case), else through the wrapped
  // coordinates.
  auto body = [&](auto inner_tag) {
    constexpr bool INNER = decltype(inner_tag)::value;
    double* const own_rec = a.dst + uint64_t(n) * kQ;
    const Idx<false> I{a.P, a.nx, a.ny};
    Coords c;
    if (!INNER) fill_coords(a, x0 + tx, y0 + ty, z0 + tz, c);
    auto far = [&](int d) -> double* {
      if (INNER) return own_rec + a.odd_off[d];
      return a.dst + I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)]);
    };
    double q[kQ];
    if (!HALO && !solid) {  // entries into rows that are not staged: now, ahead of the copies
#pragma unroll
      for (int d = 0; d < kQ; ++d) {
        const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
        if (!staged(hy, hz)) q[d] = *far(d);
      }
    }
    tma::mbar_wait(bar, 0);
    if (!solid) {
#pragma unroll
      for (int d = 0; d < kQ; ++d) {
        const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
        if (staged(hy, hz)) q[d] = at(int(tx) + 2 - cx(d), hy, hz)[dslot(opp(d))];
      }
      collide(q, a.trt);
#pragma unroll
      for (int d = 0; d < kQ; ++d) {
        const int hy = int(ty) + 1 - cy(d), hz = int(tz) + 1 - cz(d);
        if (hy >= 1 && hy <= kPtY && hz >= 1 && hz <= kPtZ)
          at(int(tx) + 2 - cx(d), hy, hz)[dslot(opp(d))] = q[opp(d)];
        else
          *far(d) = q[opp(d)];
      }
    }
  };
  if (tile_inner<kPtY, kPtZ>(a, x0, y0, z0))
    body(std::true_type{});
  else
    body(std::false_type{});
  __syncthreads();
  // owned-slot write-back of the tile's own rows, one warp per row: lane l
  // handles elements i = l + 32 j (j < 12) of the row, slot i % 19 of record
  // i / 19 (records x0-2 .. x0+17).  Which of them the tile owns depends on
  // the row only through its first / last y and z position, so the lane's
  // masks are built once: bit j of kx = owner inside the tile in x, of
  // ypos / yneg / zpos / zneg = the slot's direction has c = +1 / -1.
  constexpr int kJ = kOwnJ;
  const uint32_t lane = t & 31, warp = t >> 5;
  const uint32_t mx = kOwnMasks.mx[lane], ypos = kOwnMasks.ypos[lane], yneg = kOwnMasks.yneg[lane],
                 zpos = kOwnMasks.zpos[lane], zneg = kOwnMasks.zneg[lane];
  const uint64_t nx = a.nx;
  const bool xwrap = x0 < 2 || uint64_t(x0) + kPtX + 2 > nx;
  for (uint32_t r = warp; r < uint32_t(kPtY * kPtZ); r += kT / 32) {
    const int hy = 1 + static_cast<int>(r % kPtY), hz = 1 + static_cast<int>(r / kPtY);
    // owner y = hy - c_y must stay in [1, kPtY]: the first row excludes
    // c_y = +1, the last c_y = -1 (likewise in z)
    uint32_t m = mx;
    if (hy == 1) m &= ~ypos;
    if (hy == kPtY) m &= ~yneg;
    if (hz == 1) m &= ~zpos;
    if (hz == kPtZ) m &= ~zneg;
    const double* src = sh + size_t(HALO ? hz * (kPtY + 2) + hy : (hz - 1) * kPtY + (hy - 1)) * kRowElems;
    const uint64_t y = y0 + hy - 1, z = z0 + hz - 1;  // own rows: no y / z wrap
    double* row = a.dst + (z * a.ny + y) * nx * kQ;
    if (!xwrap) {
      double* g = row + (uint64_t(x0) - 2) * kQ;
#pragma unroll
      for (int jj = 0; jj < kJ; ++jj)
        if ((m >> jj) & 1u) g[lane + 32 * jj] = src[lane + 32 * jj];
    } else {
#pragma unroll
      for (int jj = 0; jj < kJ; ++jj) {
        if (!((m >> jj) & 1u)) continue;
        const int i = static_cast<int>(lane) + 32 * jj;
        const int hx = i / kQ;
        int64_t gx = int64_t(x0) + hx - 2;
        if (gx < 0) gx += nx;
        if (gx >= int64_t(nx)) gx -= nx;
        row[uint64_t(gx) * kQ + (i - hx * kQ)] = src[i];
      }
    }
  }
}

}  // namespace lbmgpu

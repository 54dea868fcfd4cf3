// AoS list AA odd step through 3-D staging tiles (list-aa-aos, blk = 0).
// (part of the list-addressing translation unit, included by list.cu)
//
// The odd sub-step of kernels_list_aa.cpp:22-31 gathers direction d of node n
// through Scatter entry (n, opp d) and scatters it back through entry (n, d):
// 18 scattered 8-byte loads and 18 scattered 8-byte stores per node, each one
// 32-byte sector request in the AoS layout (slot 19 m + d).  Slot s of record
// m is read and written in this sub-step only by its owner node m - c_s (or
// by m itself through a bounce-back entry), so a CTA may stage whole records
// in shared memory, gather and scatter there, and write back exactly the
// slots its own nodes produced.
//
// Node order blk = 0 (order_nodes, list_lattice.cpp:127-132) is x, y, z with
// z fastest, so the fluid nodes of one box row (x, y) inside a z range are
// ONE contiguous list range: [crank(x, y, za), crank(x, y, zb)) with crank the
// exclusive scan of the fluid flags in box order.  A CTA owns a TX x TY x TZ
// box tile; it stages its own TX x TY rows -- with EDGES also the edge halo
// rows around them -- over z in [z0-1, z0+TZ] (two list ranges where the
// range wraps periodically in z) by 1-D TMA bulk copies; entries into rows
// that are not staged are read from global memory ahead of the copies and
// stored there directly (own rows only measured fastest: the halo rows'
// few needed slots cost more as staged whole records).  Every fluid node
// looks each of its 18 entries up in the staged rows (the adjacency values stay the only source of addresses:
// entry e is found in the staged list range that holds element e),
// collides, and writes results for records in the tile's own rows into the
// staged copy (marking the element), results for halo rows straight to
// global memory.  The own rows then leave by
// coalesced stores of the marked elements only.  A record that is not found
// in its expected staged row (cannot happen for a structure built by
// build_structure, but nothing depends on it) is read and written in global
// memory directly, so the result is bitwise the per-node kernel's for any
// tile shape.
#pragma once

#include "list_sweeps.cuh"
#include "tma.cuh"

namespace lbmgpu {

struct LTileGeom {
  const uint32_t* crank;  // exclusive fluid scan in box order, V + 1 entries
  uint32_t nx, ny, nz;
  uint32_t tiles_y, tiles_z;
};

// Staged list range(s) of one halo row, in ELEMENT numbers (slot e = 19 m +
// s of record m): entry e lies in the first staged range iff e - lo0 < n0,
// and then sits at shared element e + off0 (likewise lo1 / n1 / off1 for the
// second range of a periodically wrapped z range); no division by 19.
struct __align__(16) LTileRow {
  uint32_t lo0, n0, off0, g0;  // g0: first global element copied (16-byte aligned)
  uint32_t lo1, n1, off1, g1;
  uint32_t cnt0, cnt1, pad0, pad1;  // elements copied per range (even counts)
};

template <int TX, int TY, int TZ, bool EDGES = true>
struct LTileShape {
  static constexpr int kT = TX * TY * TZ;
  static constexpr int kRows = (TX + 2) * (TY + 2);  // halo rows incl. the 4 corners
  static constexpr int kStaged = EDGES ? kRows - 4 : TX * TY;  // corners (edges) not staged
  static constexpr int kInner = TX * TY;
  // two ranges' 16-byte slack; a multiple of 4 so the marks of the own rows
  // are cleared with 16-byte stores
  static constexpr int kRowElems = ((TZ + 2) * kQ + 4 + 3) / 4 * 4;
  static constexpr size_t kStageBytes = size_t(kStaged) * kRowElems * 8;
  static constexpr size_t kFlagBytes = size_t(kInner) * kRowElems;  // marks: own rows only
  static constexpr size_t kMetaBytes = size_t(kRows) * sizeof(LTileRow);
  static constexpr size_t kSmem = kStageBytes + kFlagBytes + kMetaBytes + 16;
  static_assert(kStaged * kRowElems < (1 << 14) && kInner * kRowElems < (1 << 13),
                "packed staging positions");
  static_assert(kFlagBytes % 16 == 0 && kStageBytes % 16 == 0, "alignment");
};

__device__ __forceinline__ uint32_t even_down(uint32_t v) { return v & ~1u; }
__device__ __forceinline__ uint32_t even_up(uint32_t v) { return (v + 1u) & ~1u; }

// 2 CTAs of 256 threads per SM (<= 128 registers); 4 of 128
template <int TX, int TY, int TZ, bool EDGES = true>
__global__ void __launch_bounds__(TX * TY * TZ, 512 / (TX * TY * TZ))
    k_list_aa_odd_aos_tile(const ListArgs a, const LTileGeom g) {
  using S = LTileShape<TX, TY, TZ, EDGES>;
  extern __shared__ __align__(128) unsigned char lt_smem[];
  double* sh = reinterpret_cast<double*>(lt_smem);
  uint8_t* flag = lt_smem + S::kStageBytes;
  LTileRow* meta = reinterpret_cast<LTileRow*>(lt_smem + S::kStageBytes + S::kFlagBytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(lt_smem + S::kStageBytes + S::kFlagBytes +
                                              S::kMetaBytes);
  const uint32_t t = threadIdx.x;
  auto is_corner = [](uint32_t h) {  // not staged
    const uint32_t hx = h / (TY + 2), hy = h % (TY + 2);
    const bool ex = hx == 0 || hx == TX + 1, ey = hy == 0 || hy == TY + 1;
    return EDGES ? ex && ey : ex || ey;
  };
  auto staged_row = [](uint32_t h) {  // staged halo row -> staged row
    if (!EDGES) return (h / (TY + 2) - 1) * TY + (h % (TY + 2) - 1);
    return h - (h > 0) - (h > TY + 1) - (h > (TX + 1) * (TY + 2));
  };
  // grid (z tiles, y tiles, x tiles): the launch order is z fastest, the
  // order of the list
  const uint32_t z0 = blockIdx.x * TZ, y0 = blockIdx.y * TY, x0 = blockIdx.z * TX;
  const uint32_t zend = min(z0 + TZ, g.nz);
  // global loads first, all independent: the own cell's scan entries and
  // the halo rows' range bounds (one round trip before the TMA copies and
  // the adjacency loads are issued)
  const uint32_t tz = t % TZ, ty = (t / TZ) % TY, tx = t / (TZ * TY);
  const uint32_t x = x0 + tx, y = y0 + ty, z = z0 + tz;
  const bool inbox = x < g.nx && y < g.ny && z < g.nz;
  uint32_t n = 0, n1 = 0;
  if (inbox) {
    const uint64_t c = (uint64_t(x) * g.ny + y) * g.nz + z;
    n = g.crank[c];
    n1 = g.crank[c + 1];
  }
  static_assert(S::kRows <= S::kT, "one halo row per thread");
  // halo row h = t = hx * (TY + 2) + hy  <->  box row ((x0 + hx - 1) mod nx, (y0 + hy - 1) mod ny)
  uint32_t r0 = 0, r0e = 0, r1 = 0, r1e = 0;
  if (t < uint32_t(S::kRows)) {
    const uint32_t hx = t / (TY + 2), hy = t % (TY + 2);
    const uint32_t X = (x0 + hx + g.nx - 1) % g.nx, Y = (y0 + hy + g.ny - 1) % g.ny;
    const uint64_t c0 = (uint64_t(X) * g.ny + Y) * g.nz;
    uint32_t za0, za1, zb0 = 0, zb1 = 0;
    if (TZ + 2 >= int(g.nz)) {
      za0 = 0;
      za1 = g.nz;
    } else if (z0 == 0) {
      za0 = g.nz - 1;
      za1 = g.nz;
      zb1 = zend + 1;
    } else if (zend == g.nz) {
      za0 = z0 - 1;
      za1 = g.nz;
      zb1 = 1;
    } else {
      za0 = z0 - 1;
      za1 = zend + 1;
    }
    r0 = g.crank[c0 + za0];
    r0e = g.crank[c0 + za1];
    r1 = g.crank[c0 + zb0];
    r1e = g.crank[c0 + zb1];
  }
  if (t == 0) {
    tma::mbar_init(bar, S::kRows);
    tma::fence_barrier_init();
  }
  {  // clear the written-element marks of the own rows
    uint4* f16 = reinterpret_cast<uint4*>(flag);
    for (uint32_t i = t; i < S::kFlagBytes / 16; i += S::kT) f16[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (t < uint32_t(S::kRows)) {
    // staged row of halo row t: the corner rows (x0-1 / x0+TX, y0-1 / y0+TY)
    // are not staged -- only the 4 corner nodes' diagonal entries point
    // there, and those go to global memory -- so rows after a corner move
    // up by one
    const bool corner = is_corner(t);
    if (corner) r0 = r0e = r1 = r1e = 0;
    const uint32_t base = staged_row(t) * S::kRowElems;
    LTileRow m;
    m.lo0 = r0 * kQ;
    m.n0 = (r0e - r0) * kQ;
    m.g0 = even_down(m.lo0);
    m.cnt0 = m.n0 ? even_up(m.lo0 + m.n0) - m.g0 : 0u;
    m.off0 = base - m.g0;
    m.lo1 = r1 * kQ;
    m.n1 = (r1e - r1) * kQ;
    m.g1 = even_down(m.lo1);
    m.cnt1 = m.n1 ? even_up(m.lo1 + m.n1) - m.g1 : 0u;
    m.off1 = base + m.cnt0 - m.g1;
    meta[t] = m;
    tma::mbar_arrive_expect_tx(bar, (m.cnt0 + m.cnt1) * 8u);
    double* dst = sh + base;
    if (m.cnt0) tma::bulk_g2s(dst, a.dst + m.g0, m.cnt0 * 8u, bar);
    if (m.cnt1) tma::bulk_g2s(dst + m.cnt0, a.dst + m.g1, m.cnt1 * 8u, bar);
  }
  const bool fluid = inbox && n1 != n;
  uint32_t e[18];
  if (fluid) {
#pragma unroll
    for (int k = 1; k < kQ; ++k) e[k - 1] = __ldg(a.adj + (k - 1) * a.N + n);
  }
  __syncthreads();  // meta visible
  // packed position of an entry: staged element | (mark index << 14) when the
  // record lies in one of the tile's own rows; staged element | kDirect for a
  // halo row (the result is stored straight to global memory); kMiss = not
  // staged (read and written in global memory).
  constexpr uint32_t kDirect = 0x80000000u, kMiss = 0xffffffffu, kPos = (1u << 14) - 1;
  // own row h_i = (hx, hy) = (i / TY + 1, i % TY + 1), staged at row h - 2
  // (two corners before it), has mark rows at i * kRowElems:
  // mark index = staged element - (2 hx + TY - 1) * kRowElems
  auto mark_delta = [](uint32_t h) -> uint32_t {
    const uint32_t hx = h / (TY + 2);
    return EDGES ? (2 * hx + TY - 1) * S::kRowElems : 0u;
  };
  // generic lookup: the row's first range, its second range, else kMiss
  auto lookup = [&](uint32_t h, uint32_t v) -> uint32_t {
    const LTileRow& m = meta[h];
    if (v - m.lo0 < m.n0) return v + m.off0;
    if (v - m.lo1 < m.n1) return v + m.off1;
    return kMiss;
  };
  const uint32_t hown = (tx + 1) * (TY + 2) + (ty + 1);
  uint32_t pos[18];
  uint32_t pos0 = 0;
  bool slow = false;  // some entry needs the generic lookup
  if (fluid) {
    {
      const uint4 m0 = *reinterpret_cast<const uint4*>(&meta[hown]);
      const uint32_t v = n * kQ;
      pos0 = v - m0.x < m0.y ? v + m0.z : lookup(hown, v);
      if (pos0 != kMiss) pos0 |= (pos0 - mark_delta(hown)) << 14;
    }
#pragma unroll
    for (int k = 1; k < kQ; ++k) {
      // record n + c_k (fluid neighbour): the first staged range of row h
      const uint32_t h = hown + uint32_t(cx(k) * (TY + 2) + cy(k));
      const bool inx = uint32_t(int(tx) + cx(k)) < uint32_t(TX);
      const bool iny = uint32_t(int(ty) + cy(k)) < uint32_t(TY);
      if (EDGES ? !inx && !iny : !inx || !iny) {  // not staged (or bounce-back): global memory
        pos[k - 1] = kMiss;
        continue;
      }
      const uint4 m0 = *reinterpret_cast<const uint4*>(&meta[h]);
      const uint32_t v = e[k - 1];
      const uint32_t p = v + m0.z;
      slow |= !(v - m0.x < m0.y);
      pos[k - 1] = inx && iny ? (p | ((p - mark_delta(h)) << 14)) : (p | kDirect);
    }
    if (slow) {  // second ranges (periodic z wrap), bounce-back entries, misses
#pragma unroll
      for (int k = 1; k < kQ; ++k) {
        uint32_t h = hown + uint32_t(cx(k) * (TY + 2) + cy(k));
        const bool inx = uint32_t(int(tx) + cx(k)) < uint32_t(TX);
        const bool iny = uint32_t(int(ty) + cy(k)) < uint32_t(TY);
        if (EDGES ? !inx && !iny : !inx || !iny) continue;  // kMiss from the fast path
        bool inner = inx && iny;
        uint32_t p = lookup(h, e[k - 1]);
        if (p == kMiss) {  // bounce-back closure: the node's own record
          h = hown;
          inner = true;
          p = lookup(hown, e[k - 1]);
        }
        if (p != kMiss) p = inner ? (p | ((p - mark_delta(h)) << 14)) : (p | kDirect);
        pos[k - 1] = p;
      }
    }
  }
  // entries outside the staged rows (corner directions, misses): read now,
  // ahead of the copies
  double q[kQ];
  if (fluid) {
    if (pos0 == kMiss) q[0] = a.dst[uint64_t(n) * kQ];
#pragma unroll
    for (int d = 1; d < kQ; ++d)
      if (pos[opp(d) - 1] == kMiss) q[d] = a.dst[e[opp(d) - 1]];
  }
  tma::mbar_wait(bar, 0);
  if (fluid) {
    if (pos0 != kMiss) q[0] = sh[pos0 & kPos];
#pragma unroll
    for (int d = 1; d < kQ; ++d) {
      const uint32_t p = pos[opp(d) - 1];
      if (p != kMiss) q[d] = sh[p & kPos];
    }
    collide(q, a.trt);
    if (pos0 != kMiss) {
      sh[pos0 & kPos] = q[0];
      flag[pos0 >> 14] = 1;
    } else {
      a.dst[uint64_t(n) * kQ] = q[0];
    }
#pragma unroll
    for (int d = 1; d < kQ; ++d) {
      const uint32_t p = pos[d - 1];
      if (p & kDirect) {
        a.dst[e[d - 1]] = q[d];
      } else {
        sh[p & kPos] = q[d];
        flag[p >> 14] = 1;
      }
    }
  }
  __syncthreads();
  // write-back of the own rows: marked elements only, one element per lane
  // (a warp instruction covers 256 contiguous bytes)
  const uint32_t lane = t & 31, warp = t >> 5;
  for (uint32_t i = warp; i < uint32_t(S::kInner); i += S::kT / 32) {
    const uint32_t h = (i / TY + 1) * (TY + 2) + (i % TY + 1);
    const LTileRow& m = meta[h];
    const uint32_t cnt0 = m.cnt0, cnt = m.cnt0 + m.cnt1;
    const double* src = sh + staged_row(h) * S::kRowElems;
    const uint8_t* fr = flag + i * S::kRowElems;
    double* g0 = a.dst + m.g0;
    if (m.cnt1 == 0) {  // one list range (every row but those of a periodic z wrap)
#pragma unroll
      for (int it = 0; it < (S::kRowElems + 31) / 32; ++it) {
        const uint32_t j = lane + 32u * it;
        if (j < cnt0 && fr[j]) g0[j] = src[j];
      }
    } else {
      double* g1 = a.dst + m.g1 - cnt0;
#pragma unroll
      for (int it = 0; it < (S::kRowElems + 31) / 32; ++it) {
        const uint32_t j = lane + 32u * it;
        if (j < cnt && fr[j]) (j < cnt0 ? g0 : g1)[j] = src[j];
      }
    }
  }
}

}  // namespace lbmgpu

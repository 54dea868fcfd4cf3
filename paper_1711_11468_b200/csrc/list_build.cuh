// List lattices: structure construction (node order, adjacency) and the init / canonical-transfer / mass kernels.
// (part of the list-addressing translation unit, included by list.cu)
#pragma once

#include "list_sweeps.cuh"

namespace lbmgpu {

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
  // contiguous copy of the fluid populations (pads excluded) of nodes
  // [nb, ne) for the compensated sum
  const uint64_t cnt = a.ne - a.nb;
  for (uint64_t n = a.nb + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < a.ne;
       n += uint64_t(gridDim.x) * blockDim.x)
#pragma unroll
    for (int d = 0; d < kQ; ++d) out[d * cnt + (n - a.nb)] = buf[lslot<SOA>(a, n, d)];
}

}  // namespace lbmgpu

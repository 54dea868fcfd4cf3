// List AA node-range decomposition: links, local numbering, exchanges.
// (part of the list-addressing translation unit, included by list.cu)
#pragma once

#include "list_sweeps.cuh"

namespace lbmgpu {

// ---- node-range decomposition of list AA (multi-GPU) ----
// Part p owns the contiguous list nodes [n0_p, n1_p) (blk = 0: x-major, so
// parts are x-slabs) and holds only its own slots plus ghost copies of the
// remote slots its nodes' scatter entries point to, in a local numbering:
//   own slot (node n, direction slot d):  SoA d * nloc + (n - n0),
//                                         AoS (n - n0) * 19 + d
//   ghost slots:                          19 * nloc + gofs[s] + k
// where k is the rank of the global slot in the sorted list of link (p <- s)
// = the slots of s's nodes that p's entries point to.  The part's adjacency
// is remapped to local indices (boundary adjacency remap), so its sweeps are
// the single-lattice kernels on an nloc-node lattice.  Every slot is
// referenced by exactly one node, so p's odd step is the only reader/writer
// of a link's slots in that sub-step.  Exchange per AA pair: phase 0 (after
// even) s -> r, phase 1 (after odd) r -> s, of exactly these slots -- the
// list analogue of the direct z-slab plan (halo.hpp).

// node owning the slot that entry (n, column d) points to (SlotMap::slot,
// list_lattice.hpp:66-75: a fluid neighbour's slot d, else n's own opp slot)
__device__ __forceinline__ uint64_t entry_owner(const ListArgs& a, int soa, uint64_t n, int d,
                                                uint32_t e) {
  if (soa) {
    const uint64_t s = a.starts[d];
    return (e >= s && e < s + a.N) ? e - s : n;
  }
  return e / kQ;
}

// (owner node, direction slot) of a global slot
__device__ __forceinline__ void slot_node(const ListArgs& a, int soa, uint32_t e, uint64_t& m,
                                          int& dd) {
  if (!soa) {
    m = e / kQ;
    dd = static_cast<int>(e - m * kQ);
    return;
  }
  dd = 0;
#pragma unroll
  for (int d = 1; d < kQ; ++d)
    if (e >= a.starts[d]) dd = d;  // starts ascend (padding_offsets)
  m = e - a.starts[dd];
}

__device__ __forceinline__ uint64_t local_own(int soa, uint64_t m, int dd, uint64_t n0,
                                              uint64_t nloc) {
  return soa ? uint64_t(dd) * nloc + (m - n0) : (m - n0) * kQ + dd;
}

// part owning node m under the cut [N*p/P, N*(p+1)/P)
__device__ __forceinline__ int part_of_node(uint64_t m, uint64_t N, int parts) {
  int p = static_cast<int>(m * uint64_t(parts) / N);
  while (p > 0 && m < N * uint64_t(p) / parts) --p;
  while (p + 1 < parts && m >= N * uint64_t(p + 1) / parts) ++p;
  return p;
}

__global__ void k_link_flags(const ListArgs a, int soa, uint64_t nb, uint64_t ne, uint64_t olo,
                             uint64_t ohi, uint8_t* __restrict__ flags,
                             uint32_t* __restrict__ vals) {
  const uint64_t cnt = ne - nb;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt * 18;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(i / cnt) + 1;
    const uint64_t n = nb + (i - uint64_t(d - 1) * cnt);
    const uint32_t e = a.adj[uint64_t(d - 1) * a.N + n];
    const uint64_t m = entry_owner(a, soa, n, d, e);
    flags[i] = m >= olo && m < ohi;
    vals[i] = e;
  }
}

// Local adjacency of part [n0, n0 + nloc): own entries -> local own index,
// remote entries -> ghost index (binary search in the sorted link list).
__global__ void k_local_adj(const ListArgs g, int soa, uint64_t n0, uint64_t nloc, int parts,
                            const uint32_t* __restrict__ gslots,
                            const uint64_t* __restrict__ gofs, const uint64_t* __restrict__ gcnt,
                            uint32_t* __restrict__ ladj) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nloc * 18;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(i / nloc) + 1;
    const uint64_t j = i - uint64_t(d - 1) * nloc, n = n0 + j;
    const uint32_t e = g.adj[uint64_t(d - 1) * g.N + n];
    const uint64_t m = entry_owner(g, soa, n, d, e);
    uint64_t loc;
    if (m >= n0 && m < n0 + nloc) {
      uint64_t mm;
      int dd;
      slot_node(g, soa, e, mm, dd);
      loc = local_own(soa, mm, dd, n0, nloc);
    } else {
      const int s = part_of_node(m, g.N, parts);
      const uint32_t* l = gslots + gofs[s];
      uint64_t lo = 0, hi = gcnt[s];
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (l[mid] < e) lo = mid + 1; else hi = mid;
      }
      loc = nloc * kQ + gofs[s] + lo;
    }
    ladj[i] = static_cast<uint32_t>(loc);
  }
}

// local own index of each (global) slot of a link, on the owning part
__global__ void k_own_local_idx(const ListArgs g, int soa, uint64_t n0, uint64_t nloc,
                                const uint32_t* __restrict__ slots, uint64_t cnt,
                                uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t m;
    int dd;
    slot_node(g, soa, slots[i], m, dd);
    out[i] = static_cast<uint32_t>(local_own(soa, m, dd, n0, nloc));
  }
}

// initial local array of a part from the global one: own slots, then ghosts
__global__ void k_local_init(const ListArgs g, int soa, const double* __restrict__ gbuf,
                             uint64_t n0, uint64_t nloc, const uint32_t* __restrict__ gslots,
                             uint64_t nghost, double* __restrict__ lbuf) {
  const uint64_t own = nloc * kQ;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < own + nghost;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i < own) {
      const uint64_t j = soa ? i % nloc : i / kQ;
      const int d = static_cast<int>(soa ? i / nloc : i % kQ);
      lbuf[i] = soa ? gbuf[g.starts[d] + n0 + j] : gbuf[(n0 + j) * kQ + d];
    } else {
      lbuf[i] = gbuf[gslots[i - own]];
    }
  }
}

// boundary nodes of a part: any local entry in the ghost range
__global__ void k_ghost_mask(const uint32_t* __restrict__ ladj, uint64_t nloc,
                             uint8_t* __restrict__ mask) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < nloc;
       j += uint64_t(gridDim.x) * blockDim.x) {
    bool ghost = false;
    for (int d = 0; d < 18 && !ghost; ++d) ghost = ladj[uint64_t(d) * nloc + j] >= nloc * kQ;
    mask[j] = ghost;
  }
}

// link transfers: gather by index / scatter by index / indexed copy
__global__ void k_slots_pack(const uint32_t* __restrict__ idx, uint64_t cnt,
                             const double* __restrict__ buf, double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = buf[idx[i]];
}

__global__ void k_slots_unpack(const uint32_t* __restrict__ idx, uint64_t cnt,
                               const double* __restrict__ in, double* __restrict__ buf) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
       i += uint64_t(gridDim.x) * blockDim.x)
    buf[idx[i]] = in[i];
}

}  // namespace lbmgpu

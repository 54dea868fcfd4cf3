// Temporal blocking of the AA pattern (experimental, LBMGPU_AA_TB=W,G):
// one AA pair per DRAM pass for lattices far larger than L2.
// (part of the direct-addressing translation unit, included by direct.cu)
//
// The box is cut into y-bands of W rows, processed one after the other;
// inside a band a z-wavefront runs the pair with the odd sub-step G + 1
// planes behind the even one.  Wavefront step t of band b:
//   even on planes [tG, tG + G)          x rows [bW, bW + W)
//   odd  on planes [tG - G - 1, tG - 1)  x rows [bW - 1, bW + W - 1)
// (last band's odd rows run to ny), then a grid barrier.  Why this is the
// single-sweep result bit for bit (same per-node bodies, same inputs):
//  * z: odd on plane p needs even on p-1..p+1, all in earlier steps; the
//    concurrent even planes (>= tG) and odd planes (<= tG - 2, touching
//    <= tG - 1) are disjoint.
//  * y: the odd rows are skewed one row down, so an odd node at a band's
//    first row finds its lower neighbours' even results in the previous
//    band, and no node is advanced past a sub-step its neighbour still
//    needs (each slot is touched by one node per sub-step, kernels_full_
//    aa.cpp:83-92).  This needs no y wrap: only geometries whose extreme
//    rows and planes are solid (channel, pipe) -- checked on the host.
// Live set per step: about (2G + 2) plane-rows of W rows x nx, kept in L2
// between the pair's two touches of a node; the PDFs cross DRAM once per
// pair instead of twice.
#pragma once

#include "direct_fused.cuh"

namespace lbmgpu {

// Row counts of a band's even / odd ranges take four values (W, W - 1 for the
// first band's odd rows, and the last band's two); their fast divisors come
// from the host.
struct TbDivs {
  FastDiv w, wm1, last_e, last_o;
};

template <int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_full_aa_tb(DirectArgs a, uint32_t W, uint32_t G,
                                                          long pairs, TbDivs dv, GridBarrier bar) {
  const uint32_t nx = a.nx, ny = a.ny, nz = a.nzl;
  const uint32_t nb = (ny + W - 1) / W;
  const uint32_t T = (nz + 1 + G - 1) / G + 1;  // steps per band
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t G_all = gridDim.x * blockDim.x;
  for (long pr = 0; pr < pairs; ++pr) {
    for (uint32_t b = 0; b < nb; ++b) {
      const bool first = b == 0, last = b + 1 == nb;
      const uint32_t ye0 = b * W, ye1 = min(ny, ye0 + W);
      const uint32_t yo0 = first ? 0u : ye0 - 1;
      const uint32_t yo1 = last ? ny : ye1 - 1;
      const FastDiv fe = last ? dv.last_e : dv.w;
      const FastDiv fo = last ? dv.last_o : first ? dv.wm1 : dv.w;
      for (uint32_t t = 0; t < T; ++t) {
        const uint32_t pe0 = min(nz, t * G), pe1 = min(nz, t * G + G);
        const int po0i = int(t * G) - int(G) - 1, po1i = int(t * G) - 1;
        const uint32_t po0 = uint32_t(max(0, po0i)), po1 = uint32_t(max(0, min(int(nz), po1i)));
        const uint32_t ce = (pe1 - pe0) * (ye1 - ye0) * nx;
        const uint32_t co = po1 > po0 ? (po1 - po0) * (yo1 - yo0) * nx : 0;
        for (uint32_t i = tid; i < ce + co; i += G_all) {
          const bool even = i < ce;
          const uint32_t j = even ? i : i - ce;
          const uint32_t r = a.fdx.div(j);
          const uint32_t x = j - r * nx;
          const uint32_t rows = even ? ye1 - ye0 : yo1 - yo0;
          const uint32_t zr = even ? fe.div(r) : fo.div(r);
          const uint32_t y = (even ? ye0 : yo0) + (r - zr * rows);
          const uint32_t z = (even ? pe0 : po0) + zr;
          const uint32_t n = (z * ny + y) * nx + x;
          Coords c;
          decode_node(a, n, c);
          if (even)
            aa_even_node<true, false, true>(a, c, n);
          else
            aa_odd_node<true, false, true>(a, c, n);
        }
        grid_sync(bar);
      }
    }
  }
}

}  // namespace lbmgpu

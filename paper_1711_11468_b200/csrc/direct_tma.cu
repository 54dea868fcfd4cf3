// TMA-staged AA sweeps for the direct SoA lattice (aa-soa, aa-vec-soa).
//
// The register kernels in direct.cu are latency bound (ncu: long-scoreboard
// stalls dominate; 126 registers -> 16 warps/SM keep ~78 KB/SM in flight only
// while they are in their load phase).  Here a persistent CTA streams row
// tiles of T nodes through a STAGES-deep shared-memory ring filled by
// cp.async.bulk (1-D TMA) copies completing on mbarriers, so the bytes in
// flight per SM no longer depend on how many warps are resident:
//   stage = 19 direction segments of the tile (even: own row; odd: the 9
//   source rows (y-cy, z-cz), each segment widened to [x0-2, x0+T+2) so the
//   +-1 x shift of the gather is served from shared memory).
// Elements that wrap around the periodic x axis (first/last tile of a row)
// are read directly from global memory by the two edge threads.
// Stores go straight from registers (coalesced st.global).
//
// Race-freedom is the register kernels' argument: in each AA sub-step every
// slot is read and written by exactly one node (kernels_list_aa.cpp:18-20,
// kernels_full_aa.cpp:63-94), so the halo elements a tile stages but does not
// own are never used, and the elements it uses are written only by itself.
#include <cstring>

#include "direct_args.cuh"
#include "tma.cuh"

namespace lbmgpu {


template <int T, bool ODD>
struct TmaShape {
  static constexpr int W = ODD ? T + 4 : T;  // doubles per direction segment
  // 19 direction segments + the tile's T flag bytes (staged too: a plain
  // load of the flags would put one full memory latency on every tile)
  static constexpr int kStageDoubles = kQ * W + T / 8;
};

template <int T, int STAGES, bool ODD, bool CS, int MINB>
__global__ void __launch_bounds__(T, MINB) k_full_aa_tma(const DirectArgs a) {
  using S = TmaShape<T, ODD>;
  constexpr int W = S::W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sb = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + size_t(STAGES) * S::kStageDoubles * 8);
  double* buf = a.dst;
  const uint32_t tid = threadIdx.x;
  const uint32_t ntiles = a.count / T;
  const uint32_t nx = a.nx;
  const uint64_t P = a.P;

  struct Rows {
    uint32_t Y[3], Z[3], x0, z, y;
  };
  auto tile_rows = [&](uint32_t tile, Rows& r) {
    const uint32_t n0 = a.node0 + tile * T;
    const uint32_t z = a.fdP.div(n0);
    const uint32_t rem = n0 - z * a.P;
    const uint32_t y = a.fdx.div(rem);
    r.x0 = rem - y * nx;
    r.z = z;
    r.y = y;
    r.Y[0] = y == 0 ? a.ny - 1 : y - 1;
    r.Y[1] = y;
    r.Y[2] = y + 1 == a.ny ? 0 : y + 1;
    const uint32_t zs = z + a.zoff;
    if (a.zwrap) {
      r.Z[0] = z == 0 ? a.nzl - 1 : z - 1;
      r.Z[2] = z + 1 == a.nzl ? 0 : z + 1;
    } else {
      r.Z[0] = zs - 1;
      r.Z[2] = zs + 1;
    }
    r.Z[1] = zs;
  };
  auto row_ptr = [&](uint32_t zs, int slot, uint32_t y) -> double* {
    return buf + (uint64_t(zs) * kQ + slot) * P + uint64_t(y) * nx;
  };

  // thread 0: stage the tile's 19 segments into ring slot s
  auto issue = [&](uint32_t tile, int s) {
    Rows r;
    tile_rows(tile, r);
    double* st = sb + size_t(s) * S::kStageDoubles;
    uint32_t bytes = 0;
    const void* srcs[kQ];
    uint32_t offs[kQ], lens[kQ];
#pragma unroll
    for (int d = 0; d < kQ; ++d) {
      if (!ODD) {
        srcs[d] = row_ptr(r.Z[1], dslot(d), r.y) + r.x0;
        offs[d] = 0;
        lens[d] = T;
      } else {
        const double* row = row_ptr(r.Z[1 - cz(d)], dslot(opp(d)), r.Y[1 - cy(d)]);
        if (d == 0 || cx(d) == 0) {
          srcs[d] = row + r.x0;
          offs[d] = 2;
          lens[d] = T;
        } else {
          const int lo = max(int(r.x0) - 2, 0);
          const int hi = min(int(r.x0) + T + 2, int(nx));
          srcs[d] = row + lo;
          offs[d] = static_cast<uint32_t>(lo - (int(r.x0) - 2));
          lens[d] = static_cast<uint32_t>(hi - lo);
        }
      }
      bytes += lens[d] * 8;
    }
    tma::fence_proxy_async();
    tma::mbar_arrive_expect_tx(&bars[s], bytes + T);
#pragma unroll
    for (int d = 0; d < kQ; ++d)
      tma::bulk_g2s(st + d * W + offs[d], srcs[d], lens[d] * 8, &bars[s]);
    tma::bulk_g2s(st + kQ * W, a.flags + a.node0 + tile * T, T, &bars[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) {
      const uint32_t tile = blockIdx.x + s * gridDim.x;
      if (tile < ntiles) issue(tile, s);
    }

  uint32_t it = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = static_cast<int>(it % STAGES);
    Rows r;
    tile_rows(tile, r);
    const uint32_t x = r.x0 + tid;
    tma::mbar_wait(&bars[s], (it / STAGES) & 1);
    const double* st = sb + size_t(s) * S::kStageDoubles;
    const bool fluid = reinterpret_cast<const uint8_t*>(st + kQ * W)[tid] == 0;
    if (fluid) {
      double q[kQ];
      if (!ODD) {
#pragma unroll
        for (int d = 0; d < kQ; ++d) q[d] = st[d * W + tid];
        collide(q, a.trt);
        const uint64_t own = uint64_t(r.Z[1]) * kQ * P + uint64_t(r.y) * nx + x;
#pragma unroll
        for (int d = 0; d < kQ; ++d) {
          double* p = buf + own + uint64_t(dslot(opp(d))) * P;
          if (CS) __stcs(p, q[d]); else *p = q[d];
        }
      } else {
#pragma unroll
        for (int d = 0; d < kQ; ++d) {
          const int xs = int(x) - cx(d);
          if (xs >= 0 && xs < int(nx)) {
            q[d] = st[d * W + tid + 2 - cx(d)];
          } else {  // periodic x wrap: read the other end of the row
            const uint32_t xw = xs < 0 ? nx - 1 : 0;
            q[d] = row_ptr(r.Z[1 - cz(d)], dslot(opp(d)), r.Y[1 - cy(d)])[xw];
          }
        }
        collide(q, a.trt);
        const uint32_t X[3] = {x == 0 ? nx - 1 : x - 1, x, x + 1 == nx ? 0 : x + 1};
#pragma unroll
        for (int d = 0; d < kQ; ++d) {
          double* p = row_ptr(r.Z[1 + cz(d)], dslot(d), r.Y[1 + cy(d)]) + X[1 + cx(d)];
          if (CS) __stcs(p, q[d]); else *p = q[d];
        }
      }
    }
    __syncthreads();  // ring slot s fully consumed
    if (tid == 0) {
      const uint32_t next = tile + STAGES * gridDim.x;
      if (next < ntiles) issue(next, s);
    }
  }
}

template <int T, int STAGES, bool ODD, bool CS, int MINB>
static bool launch_one(const DirectArgs& a, int sm_count, cudaStream_t s) {
  using S = TmaShape<T, ODD>;
  const size_t smem = size_t(STAGES) * S::kStageDoubles * 8 + STAGES * 8;
  static bool configured = false;
  if (!configured) {
    LBM_CUDA(cudaFuncSetAttribute(k_full_aa_tma<T, STAGES, ODD, CS, MINB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = true;
  }
  const uint32_t ntiles = a.count / T;
  const int grid = static_cast<int>(std::min<uint32_t>(ntiles, uint32_t(sm_count) * MINB));
  k_full_aa_tma<T, STAGES, ODD, CS, MINB><<<grid, T, smem, s>>>(a);
  LBM_CHECK_LAUNCH();
  return true;
}

template <int STAGES, int MINB>
static bool launch_pair(bool odd, const DirectArgs& a, int sm_count, cudaStream_t s) {
  return odd ? launch_one<kTmaTile, STAGES, true, false, MINB>(a, sm_count, s)
             : launch_one<kTmaTile, STAGES, false, false, MINB>(a, sm_count, s);
}

// Returns false when the shape does not fit the tiled kernel (caller falls
// back to the register kernels).  T must divide nx; nx even keeps every
// staged segment 16-byte aligned.  config = stages + 10*(CTAs per SM - 1):
// 3, 4, 5 (one CTA per SM) or 12 (two CTAs per SM, two stages each).
bool launch_aa_tma(bool odd, const DirectArgs& a, int sm_count, int config,
                   cudaStream_t s) {
  constexpr int T = kTmaTile;
  if (a.nx % T != 0 || a.count % T != 0 || a.node0 % T != 0 || a.count == 0) return false;
  switch (config) {
    case 3: return launch_pair<3, 1>(odd, a, sm_count, s);
    case 5: return launch_pair<5, 1>(odd, a, sm_count, s);
    case 12: return launch_pair<2, 2>(odd, a, sm_count, s);
    default: return launch_pair<4, 1>(odd, a, sm_count, s);
  }
}

}  // namespace lbmgpu

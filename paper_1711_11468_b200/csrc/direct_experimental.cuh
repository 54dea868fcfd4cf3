// Measured-slower sweep variants kept opt-in for reproduction.
// (part of the direct-addressing translation unit, included by direct.cu)
#pragma once

#include "direct_args.cuh"
#include "direct_node.cuh"

namespace lbmgpu {

// Odd step with the x-shifted scatters realigned through shared memory.
// In k_full_aa_odd every warp stores the 10 directions with c_x != 0 one
// element off its own x range, so each such store instruction writes two
// partial 32-byte sectors (one shared with the neighbouring warp).  Here a
// 128-thread block covers 128 consecutive x of one row (nx % 128 == 0): the
// producer of the value that lands on x_u parks it in shared memory, and
// thread u stores it aligned; only the two elements that leave the block's x
// range are stored by their producers directly.  Loads, collision and the
// order of values are unchanged, so results are bitwise those of
// k_full_aa_odd.
constexpr int kSxThreads = 128;
template <int MINB>
__global__ void __launch_bounds__(kSxThreads, MINB) k_full_aa_odd_sx(const DirectArgs a) {
  constexpr int kX = 10;  // directions with c_x != 0
  __shared__ double sh[kX][kSxThreads];
  __shared__ uint8_t fl[kSxThreads];
  const int u = threadIdx.x;
  const uint32_t n = a.node0 + blockIdx.x * kSxThreads + u;
  Coords c;
  decode_node(a, n, c);
  const bool fluid = !solid_node(a, c.x, c.y, c.z, n);
  fl[u] = fluid;
  const Idx<true> I{a.P, a.nx, a.ny};
  double* buf = a.dst;
  if (fluid) {
    // gather/scatter address of direction d: own slot-0 element + constant
    // for interior warps (see aa_odd_node), the wrapped form otherwise
    const bool inner = c.x - 1u < a.nx - 2u && c.y - 1u < a.ny - 2u &&
                       (!a.zwrap || c.z - 1u < a.nzl - 2u);
    const bool fast = __all_sync(__activemask(), inner);
    double* own = buf + I(c.Z[1], 0, c.y, c.x);
    auto addr = [&](int d) -> double* {
      if (fast) return own + a.odd_off[d];
      return d == 0 ? buf + I(c.Z[1], dslot(0), c.y, c.x)
                    : buf + I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)]);
    };
    double q[kQ];
#pragma unroll
    for (int d = 0; d < kQ; ++d) q[d] = *addr(d);
    collide(q, a.trt);
    int k = 0;
#pragma unroll
    for (int d = 0; d < kQ; ++d) {
      if (cx(d) == 0) {
        *addr(d) = q[opp(d)];
      } else {
        const int dst = u - cx(d);  // the thread whose x the value lands on
        if (dst >= 0 && dst < kSxThreads)
          sh[k][dst] = q[opp(d)];
        else
          *addr(d) = q[opp(d)];
        ++k;
      }
    }
  }
  __syncthreads();
  int k = 0;
#pragma unroll
  for (int d = 1; d < kQ; ++d) {
    if (cx(d) == 0) continue;
    const int src = u + cx(d);
    if (src >= 0 && src < kSxThreads && fl[src])
      buf[I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.x)] = sh[k][u];
    ++k;
  }
}

// ---- AA sub-steps, software-pipelined through shared memory ---------------
// Persistent variant of k_full_aa_even / k_full_aa_odd (direct_node.cuh).  Each thread walks nodes
// n, n + G, n + 2G, ... (G = grid size) and, while it collides node n, the
// 19 populations of its next node are already in flight as per-thread
// cp.async (LDGSTS) copies into its own shared-memory column: the load
// latency of node n+G overlaps the collision of node n inside every warp
// instead of depending on other resident warps.  Each thread only ever
// reads the shared-memory slots it filled itself, so no block barrier is
// needed -- cp.async.wait_group orders it.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


// Address of the slot a node gathers direction d from (odd: (x - c_d, opp d);
// even: (x, d)); in the odd step it is also where direction opp(d) is stored.
template <bool ODD>
__device__ __forceinline__ uint64_t aa_src(const Idx<true>& I, const Coords& c, int d) {
  if (ODD && d != 0)
    return I(c.Z[1 - cz(d)], dslot(opp(d)), c.Y[1 - cy(d)], c.X[1 - cx(d)]);
  return I(c.Z[1], dslot(d), c.y, c.x);
}

constexpr int kPipeThreads = 256;

template <bool ODD, int STAGES, int MINB>
__global__ void __launch_bounds__(kPipeThreads, MINB) k_full_aa_pipe(const DirectArgs a) {
  extern __shared__ double sm_pipe[];  // [STAGES][19][kPipeThreads]
  const uint32_t tid = threadIdx.x;
  const uint32_t G = gridDim.x * kPipeThreads;
  const uint32_t end = a.node0 + a.count;
  const Idx<true> I{a.P, a.nx, a.ny};
  double* buf = a.dst;
  uint8_t solid[STAGES];
  auto prefetch = [&](uint32_t n, int s) {
    if (n < end) {
      Coords c;
      decode_node(a, n, c);
      solid[s] = a.flags[n];
      double* col = sm_pipe + size_t(s) * kQ * kPipeThreads + tid;
#pragma unroll
      for (int d = 0; d < kQ; ++d) cp_async8(col + d * kPipeThreads, buf + aa_src<ODD>(I, c, d));
    }
    cp_async_commit();
  };
  uint32_t n = a.node0 + blockIdx.x * kPipeThreads + tid;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) prefetch(n + s * G, s);
  while (n < end) {
    // unrolled by STAGES so the ring index (and solid[]) is a constant
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      if (n < end) {
        prefetch(n + (STAGES - 1) * G, (s + STAGES - 1) % STAGES);
        cp_async_wait<STAGES - 1>();
        if (!solid[s]) {
          const double* col = sm_pipe + size_t(s) * kQ * kPipeThreads + tid;
          double q[kQ];
#pragma unroll
          for (int d = 0; d < kQ; ++d) q[d] = col[d * kPipeThreads];
          collide(q, a.trt);
          Coords c;
          decode_node(a, n, c);
          if (ODD) {
#pragma unroll
            for (int d = 0; d < kQ; ++d) buf[aa_src<true>(I, c, d)] = q[opp(d)];
          } else {
#pragma unroll
            for (int d = 0; d < kQ; ++d) buf[I(c.Z[1], dslot(opp(d)), c.y, c.x)] = q[d];
          }
        }
        n += G;
      }
    }
  }
  cp_async_wait<0>();
}

template <bool ODD, int STAGES, int MINB>
void launch_aa_pipe(const DirectArgs& a, int sm_count, cudaStream_t s) {
  const size_t smem = size_t(STAGES) * kQ * kPipeThreads * sizeof(double);
  static bool configured = false;
  if (!configured) {
    LBM_CUDA(cudaFuncSetAttribute(k_full_aa_pipe<ODD, STAGES, MINB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = true;
  }
  const uint64_t blocks = ceil_div(a.count, kPipeThreads);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(blocks, uint64_t(sm_count) * MINB));
  k_full_aa_pipe<ODD, STAGES, MINB><<<grid, kPipeThreads, smem, s>>>(a);
  LBM_CHECK_LAUNCH();
}

}  // namespace lbmgpu

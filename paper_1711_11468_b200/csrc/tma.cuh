// 1-D TMA (cp.async.bulk) and mbarrier helpers shared by the sweeps.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace lbmgpu {
namespace tma {

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace tma

namespace tma {
// shared -> global bulk store, tracked by the issuing thread's bulk groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(saddr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the shared-memory sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
}  // namespace tma

// AoS tile of T consecutive records (19 doubles each) between global and
// shared memory: one 1-D bulk copy (TMA) per direction of travel when the
// tile is full and 16-byte aligned, the element loop of aos_tile_copy
// otherwise.  Both calls are block-wide (contain __syncthreads).
template <int T>
__device__ __forceinline__ void aos_tile_load(double* sh, const double* g, uint32_t cnt,
                                              uint64_t* bar) {
  constexpr uint32_t kBytes = T * 19 * 8;
  if (cnt == T && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    if (threadIdx.x == 0) {
      tma::mbar_init(bar, 1);
      tma::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tma::mbar_arrive_expect_tx(bar, kBytes);
      tma::bulk_g2s(sh, g, kBytes, bar);
    }
    tma::mbar_wait(bar, 0);
  } else {
    aos_tile_copy<T>(sh, g, cnt);
    __syncthreads();
  }
}

template <int T>
__device__ __forceinline__ void aos_tile_store(double* g, const double* sh, uint32_t cnt) {
  constexpr uint32_t kBytes = T * 19 * 8;
  if (cnt == T && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    tma::fence_proxy_async();  // this thread's shared writes -> async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      tma::bulk_s2g(g, sh, kBytes);
      tma::bulk_commit();
      tma::bulk_wait_read0();
    }
  } else {
    __syncthreads();
    aos_tile_copy<T>(g, sh, cnt);
  }
}

}  // namespace lbmgpu

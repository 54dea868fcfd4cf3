// Shared host/device definitions of the B200 LBM sweep library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace lbmgpu {

// ---- error classes (reference include/lbm/errors.hpp:9-18) ---------------
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

#define LBM_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess)                                                 \
      throw ::lbmgpu::DeviceError(std::string(#call) + ": " +              \
                                  cudaGetErrorString(e_) + " (" __FILE__   \
                                  ":" + std::to_string(__LINE__) + ")");   \
  } while (0)

#define LBM_CHECK_LAUNCH() LBM_CUDA(cudaGetLastError())

// ---- D3Q19 stencil (reference include/lbm/d3q19.hpp:11-54) ----------------
constexpr int kQ = 19;

// Tables live inside the accessors so they are usable from device code; with
// unrolled loops the index is a compile-time constant and the lookups fold.
__host__ __device__ constexpr int cx(int d) {
  constexpr int t[kQ] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
  return t[d];
}
__host__ __device__ constexpr int cy(int d) {
  constexpr int t[kQ] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
  return t[d];
}
__host__ __device__ constexpr int cz(int d) {
  constexpr int t[kQ] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
  return t[d];
}
// opposite directions are adjacent: opp(2k-1) = 2k (d3q19.hpp:43-44)
__host__ __device__ constexpr int opp(int d) {
  return d == 0 ? 0 : ((d & 1) ? d + 1 : d - 1);
}

constexpr double kWRest = 1.0 / 3.0;
constexpr double kWAxis = 1.0 / 18.0;
constexpr double kWDiag = 1.0 / 36.0;
__host__ __device__ constexpr double weight(int d) {
  return d == 0 ? kWRest : (d <= 6 ? kWAxis : kWDiag);
}

// ---- device storage order of the 19 directions for the DIRECT lattices ----
// Directions are grouped by c_z so that, in the [z][slot][y][x] layout, the
// five c_z=-1 ("down") and the five c_z=+1 ("up") slots of one z-plane are
// each ONE contiguous block: a z-slab halo transfer is then a single copy per
// face and phase.  The canonical order is restored at snapshot time.
//   slots 0..4   : c_z = -1  {6 B, 12 BW, 13 BE, 16 BS, 17 BN}
//   slots 5..13  : c_z =  0  {0, 1, 2, 3, 4, 7, 8, 9, 10}
//   slots 14..18 : c_z = +1  {5 T, 11 TE, 14 TW, 15 TN, 18 TS}
__host__ __device__ constexpr int dslot(int d) {
  constexpr int t[kQ] = {5, 6, 7, 8, 9, 14, 0, 10, 11, 12, 13, 15, 1, 2, 16, 17, 3, 4, 18};
  return t[d];
}
__host__ __device__ constexpr int ddir(int slot) {
  constexpr int t[kQ] = {6, 12, 13, 16, 17, 0, 1, 2, 3, 4, 7, 8, 9, 10, 5, 11, 14, 15, 18};
  return t[slot];
}
constexpr int kDownSlot0 = 0;
constexpr int kUpSlot0 = 14;
constexpr int kHaloSlots = 5;

// ---- fast unsigned division by a runtime-constant divisor ------------------
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    // Granlund-Montgomery round-up method, exact for every 32-bit n.
    s = 0;
    while ((1ull << s) < div) ++s;
    m = static_cast<uint32_t>(((1ull << 32) * ((1ull << s) - div)) / div + 1);
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    const uint32_t t = __umulhi(n, m);
#else
    const uint32_t t = static_cast<uint32_t>((uint64_t(n) * m) >> 32);
#endif
    return d == 1 ? n : (t + ((n - t) >> 1)) >> (s - 1);
  }
};

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Ordering point between a node's 19 gathers and its stores in the
// stream-only (no collision) sweeps: without the collision in between,
// ptxas interleaves the first stores with the remaining loads, and a store
// that waits on a load's data then holds back the loads behind it -- two
// memory latencies per node instead of one (measured: the AoS list stream
// pass at 1.5 TB/s against 3.6 TB/s for the collide pass).  A warp sync
// is an instruction ptxas does not move memory operations across.
__device__ __forceinline__ void loads_before_stores() { __syncwarp(__activemask()); }

// ---- AoS tiles through shared memory ---------------------------------------
// A block's `cnt` consecutive AoS records (19 doubles each) are one
// contiguous range: moved between global and shared memory with 16-byte
// accesses (8-byte ones for a ragged or unaligned tile), so an own-record
// sweep issues full-sector loads and stores instead of one 32-byte sector
// request per 8-byte element.
template <int T>
__device__ __forceinline__ void aos_tile_copy(double* dst, const double* src, uint32_t cnt) {
  const uint32_t nd = cnt * kQ;
  if (cnt == T && T % 2 == 0 &&
      ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (uint32_t i = threadIdx.x; i < nd / 2; i += T) d2[i] = s2[i];
  } else {
    for (uint32_t i = threadIdx.x; i < nd; i += T) dst[i] = src[i];
  }
}

}  // namespace lbmgpu

// Device reductions for the steady-state driver and the Poiseuille check
// (reference src/harness.cpp:141-174, src/verification.cpp:75-85).
#include <algorithm>
#include <cstring>

#include "lbm.hpp"

namespace lbmgpu {

// Non-negative doubles order like their bit patterns, so a max over them is
// an atomicMax on the 64-bit pattern.
__global__ void k_velocity_change(const double* __restrict__ u,
                                  const double* __restrict__ up, uint64_t n,
                                  unsigned long long* out /* [du, u, nonfinite] */) {
  double mdu = 0.0, mu = 0.0;
  unsigned long long bad = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double a = u[i];
    if (!isfinite(a)) bad = 1;
    mdu = fmax(mdu, fabs(a - up[i]));
    mu = fmax(mu, fabs(a));
  }
  for (int o = 16; o; o >>= 1) {
    mdu = fmax(mdu, __shfl_down_sync(0xffffffffu, mdu, o));
    mu = fmax(mu, __shfl_down_sync(0xffffffffu, mu, o));
    bad |= __shfl_down_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], __double_as_longlong(mdu));
    atomicMax(&out[1], __double_as_longlong(mu));
    if (bad) atomicOr(&out[2], 1ull);
  }
}

void velocity_change(const double* u, const double* uprev, uint64_t n3,
                     double* max_du, double* max_u, bool* finite,
                     cudaStream_t s) {
  DevBuf<unsigned long long> o(3);
  LBM_CUDA(cudaMemsetAsync(o.get(), 0, 24, s));
  int dev = 0, sms = 148;
  LBM_CUDA(cudaGetDevice(&dev));
  LBM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // grid-stride: 4 CTAs per SM, no more than the data needs
  const uint64_t want = ceil_div(n3, 256);
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 4ull * sms)));
  k_velocity_change<<<grid, 256, 0, s>>>(u, uprev, n3, o.get());
  LBM_CHECK_LAUNCH();
  unsigned long long h[3];
  LBM_CUDA(cudaMemcpyAsync(h, o.get(), 24, cudaMemcpyDeviceToHost, s));
  LBM_CUDA(cudaStreamSynchronize(s));
  std::memcpy(max_du, &h[0], 8);
  std::memcpy(max_u, &h[1], 8);
  *finite = h[2] == 0;
}

// One thread per fluid layer, summing u_x over the columns in canonical
// (snapshot) order -- the reference's loop order, hence the same rounding
// (verification.cpp:75-85 sums sequentially; a tree reduction would change
// the last bits of the reported profile).  The verification slit has 64
// columns and 32 layers, so the serial loop costs microseconds.
__global__ void k_layer_sums(const double* __restrict__ u, uint64_t cols,
                             int layers, double* __restrict__ out) {
  const int kz = blockIdx.x * blockDim.x + threadIdx.x;
  if (kz >= layers) return;
  double s = 0.0;
  for (uint64_t col = 0; col < cols; ++col) s += u[3 * (col * layers + kz)];
  out[kz] = s;
}

void layer_sums(const double* u, uint64_t cols, int layers, double* out,
                cudaStream_t s) {
  k_layer_sums<<<(layers + 127) / 128, 128, 0, s>>>(u, cols, layers, out);
  LBM_CHECK_LAUNCH();
}

}  // namespace lbmgpu

// Device bandwidth micro-benchmarks -- the GPU counterparts of the
// reference's copy / copy-19 / copy-19-nt-sl / update-19 loops
// (proj/src/microbench.cpp:57-175), used as the "adjusted" roofline ceiling
// next to the measured copy peak (the paper's second ceiling, PAPER.md:471-479;
// kernel -> micro mapping of perfmodel.cpp:68-72).
//
// Accounting is GPU-native: no write allocate, so copy = 16 B/element,
// copy-19 = copy-19-nt-sl = update-19 = 19 x 16 B per element index
// (the reference's CPU accounting adds 8 B write-allocate for the plain
// copies, microbench.cpp:92-99).  The 19 streams are planes of one
// allocation, like the lattice's slot planes.
#include <algorithm>
#include <string>
#include <vector>

#include "lbm.hpp"

namespace lbmgpu {

// One 16-byte vector (2 elements) of every stream per thread, one pass of
// threads over the arrays (no grid-stride loop): the access shape that
// reaches the highest copy bandwidth on B200.
template <int S, bool CS>
__global__ void __launch_bounds__(256) k_copy_streams(const double2* __restrict__ src,
                                                      double2* __restrict__ dst,
                                                      uint64_t n2) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n2) return;
  double2 v[S];
#pragma unroll
  for (int k = 0; k < S; ++k) v[k] = src[k * n2 + i];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    if (CS)
      __stcs(dst + k * n2 + i, v[k]);
    else
      dst[k * n2 + i] = v[k];
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_update_streams(double2* __restrict__ a, uint64_t n2,
                                                        double s) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n2) return;
  double2 v[S];
#pragma unroll
  for (int k = 0; k < S; ++k) v[k] = a[k * n2 + i];
#pragma unroll
  for (int k = 0; k < S; ++k) a[k * n2 + i] = make_double2(v[k].x * s, v[k].y * s);
}

__global__ void k_fill(double* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = 1.0;
}

// Element count and accounted bytes of one pass: `gpu` is this library's
// accounting (no write allocate: 16 B per element and stream), `ref` the
// reference's CPU accounting of the same pass (microbench.cpp:92-99: the
// plain copies add 8 B write allocate per element and stream).
MicroPlan micro_plan(const std::string& kind, uint64_t working_set_bytes) {
  MicroPlan m;
  if (kind == "copy") {
    m.streams = 1;
    m.arrays = 2;
  } else if (kind == "copy-19" || kind == "copy-19-nt-sl") {
    m.streams = kQ;
    m.arrays = 2 * kQ;
  } else if (kind == "update-19") {
    m.streams = kQ;
    m.arrays = kQ;
  } else {
    throw ConfigError("unknown micro-benchmark '" + kind +
                      "' (valid: copy, copy-19, copy-19-nt-sl, update-19)");
  }
  m.n = 2 * (working_set_bytes / (uint64_t(m.arrays) * 16));  // whole double2 per stream
  m.bytes_gpu = 16ull * m.streams * m.n;
  const bool write_allocate = kind == "copy" || kind == "copy-19";
  m.bytes_ref = (write_allocate ? 24ull : 16ull) * m.streams * m.n;
  return m;
}

// Median GB/s over `reps` timed passes after one warm-up pass.
double run_microbench(const std::string& kind, uint64_t working_set_bytes, int reps) {
  const MicroPlan plan = micro_plan(kind, working_set_bytes);
  const int arrays = plan.arrays;
  int dev = 0, l2 = 0, sms = 148;
  LBM_CUDA(cudaGetDevice(&dev));
  LBM_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  LBM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (working_set_bytes < 4ull * uint64_t(l2))
    throw ConfigError("microbench: working set below 4x the L2 (" +
                      std::to_string(4ull * uint64_t(l2)) + " B)");
  if (reps < 1) throw ConfigError("microbench: reps must be >= 1");
  const uint64_t n = plan.n, n2 = n / 2;  // elements / double2 per stream
  DevBuf<double> buf(n * arrays);
  cudaStream_t s;
  LBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  k_fill<<<sms * 8, 256, 0, s>>>(buf.get(), n * arrays);
  LBM_CHECK_LAUNCH();
  const unsigned grid = static_cast<unsigned>(ceil_div(n2, 256));
  double2* b2 = reinterpret_cast<double2*>(buf.get());
  auto pass = [&] {
    if (kind == "copy")
      k_copy_streams<1, false><<<grid, 256, 0, s>>>(b2, b2 + n2, n2);
    else if (kind == "copy-19")
      k_copy_streams<kQ, false><<<grid, 256, 0, s>>>(b2, b2 + kQ * n2, n2);
    else if (kind == "copy-19-nt-sl")
      k_copy_streams<kQ, true><<<grid, 256, 0, s>>>(b2, b2 + kQ * n2, n2);
    else
      k_update_streams<kQ><<<grid, 256, 0, s>>>(b2, n2, 1.0000001);
    LBM_CHECK_LAUNCH();
  };
  cudaEvent_t a, b;
  LBM_CUDA(cudaEventCreate(&a));
  LBM_CUDA(cudaEventCreate(&b));
  pass();
  std::vector<double> gbps;
  const double bytes = double(plan.bytes_gpu);
  for (int r = 0; r < reps; ++r) {
    LBM_CUDA(cudaEventRecord(a, s));
    pass();
    LBM_CUDA(cudaEventRecord(b, s));
    LBM_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    LBM_CUDA(cudaEventElapsedTime(&ms, a, b));
    gbps.push_back(bytes / (ms / 1e3) / 1e9);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  std::sort(gbps.begin(), gbps.end());
  return gbps[gbps.size() / 2];
}

}  // namespace lbmgpu

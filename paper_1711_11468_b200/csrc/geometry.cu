// Device-resident geometry (reference src/geometry.cpp:40-117), fluid scans,
// compensated reductions and per-kernel event statistics.
#include <map>
#include <mutex>
#include <cub/cub.cuh>

#include "lbm.hpp"

namespace lbmgpu {

// One thread per box node in canonical (x*ny+y)*nz+z order.  The solid tests
// are the reference's integer tests verbatim:
//   channel geometry.cpp:48-57, slit :58-67, pipe :68-84 (with D^2 in place of
//   (min(ny,nz)-2)^2 when a diameter is given), blocks :85-104.
__global__ void k_flags(uint8_t* __restrict__ flags, int kind, int nx, int ny,
                        int nz, int block, int spacing, long long d2,
                        uint64_t V) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= V) return;
  const int z = static_cast<int>(i % nz);
  const uint64_t r = i / nz;
  const int y = static_cast<int>(r % ny);
  const int x = static_cast<int>(r / ny);
  uint8_t s = 0;
  switch (kind) {
    case kChannel:
      s = (y == 0 || y == ny - 1 || z == 0 || z == nz - 1);
      break;
    case kSlit:
      s = (z == 0 || z == nz - 1);
      break;
    case kPipe: {
      const long long dy = 2LL * y - (ny - 1);
      const long long dz = 2LL * z - (nz - 1);
      s = (dy * dy + dz * dz > d2);
      break;
    }
    case kBlocks: {
      const int p = block + spacing;
      s = (x % p >= spacing && y % p >= spacing && z % p >= spacing);
      break;
    }
  }
  flags[i] = s;
}

struct IsFluid {
  __host__ __device__ __forceinline__ uint32_t operator()(uint8_t f) const {
    return f == 0 ? 1u : 0u;
  }
};

uint64_t scan_fluid(const uint8_t* flags, uint32_t* out, uint64_t n,
                    cudaStream_t s) {
  if (n >= (1ull << 32)) throw ConfigError("scan_fluid: box too large");
  cub::TransformInputIterator<uint32_t, IsFluid, const uint8_t*> it(flags,
                                                                   IsFluid{});
  size_t tmp = 0;
  LBM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, out,
                                         static_cast<int64_t>(n), s));
  DevBuf<uint8_t> t(tmp);
  LBM_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, it, out,
                                         static_cast<int64_t>(n), s));
  uint32_t last = 0;
  uint8_t lastf = 1;
  if (n) {
    LBM_CUDA(cudaMemcpyAsync(&last, out + n - 1, 4, cudaMemcpyDeviceToHost, s));
    LBM_CUDA(cudaMemcpyAsync(&lastf, flags + n - 1, 1, cudaMemcpyDeviceToHost, s));
  }
  LBM_CUDA(cudaStreamSynchronize(s));
  return n ? uint64_t(last) + (lastf == 0) : 0;
}

DeviceGeometry build_geometry_device(const GeomSpec& g, cudaStream_t s) {
  const std::array<bool, 3> per = validate_geometry(g);
  DeviceGeometry dg;
  dg.nx = g.nx;
  dg.ny = g.ny;
  dg.nz = g.nz;
  dg.periodic = per;
  const uint64_t V = g.volume();
  dg.flags.alloc(V);
  if (g.kind == kCustom) {
    LBM_CUDA(cudaMemcpyAsync(dg.flags.get(), g.custom.data(), V,
                             cudaMemcpyHostToDevice, s));
  } else {
    long long D = g.pipe_diameter > 0 ? g.pipe_diameter
                                      : (long long)std::min(g.ny, g.nz) - 2;
    const int threads = 256;
    k_flags<<<static_cast<unsigned>(ceil_div(V, threads)), threads, 0, s>>>(
        dg.flags.get(), g.kind, g.nx, g.ny, g.nz, g.block, g.spacing, D * D, V);
    LBM_CHECK_LAUNCH();
  }
  // fluid_count (geometry.cpp:113-117)
  {
    cub::TransformInputIterator<uint32_t, IsFluid, const uint8_t*> it(
        dg.flags.get(), IsFluid{});
    DevBuf<unsigned long long> sum(1);
    size_t tmp = 0;
    auto op = cub::Sum();
    LBM_CUDA(cub::DeviceReduce::Reduce(nullptr, tmp, it, sum.get(),
                                       static_cast<int64_t>(V), op,
                                       0ull, s));
    DevBuf<uint8_t> t(tmp);
    LBM_CUDA(cub::DeviceReduce::Reduce(t.get(), tmp, it, sum.get(),
                                       static_cast<int64_t>(V), op,
                                       0ull, s));
    unsigned long long h = 0;
    LBM_CUDA(cudaMemcpyAsync(&h, sum.get(), 8, cudaMemcpyDeviceToHost, s));
    LBM_CUDA(cudaStreamSynchronize(s));
    dg.n_fluid = static_cast<int64_t>(h);
  }
  if (dg.n_fluid == 0) {
    static const char* names[] = {"channel", "slit", "pipe", "blocks", "custom"};
    throw ConfigError(std::string("geometry '") + names[g.kind] +
                      "' produced no fluid nodes");
  }
  return dg;
}

// ---- compensated (Neumaier) sum -------------------------------------------
struct KSum {
  double s, c;
};
__device__ __forceinline__ void neumaier(KSum& a, double v) {
  const double t = a.s + v;
  if (fabs(a.s) >= fabs(v))
    a.c += (a.s - t) + v;
  else
    a.c += (v - t) + a.s;
  a.s = t;
}
__device__ __forceinline__ KSum merge(KSum a, KSum b) {
  neumaier(a, b.s);
  a.c += b.c;
  return a;
}

__global__ void k_sum(const double* __restrict__ d, uint64_t n,
                      KSum* __restrict__ partial) {
  KSum acc{0.0, 0.0};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    neumaier(acc, d[i]);
  __shared__ KSum sh[32];
  for (int o = 16; o; o >>= 1) {
    KSum b{__shfl_down_sync(0xffffffffu, acc.s, o),
           __shfl_down_sync(0xffffffffu, acc.c, o)};
    acc = merge(acc, b);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : KSum{0.0, 0.0};
    for (int o = 16; o; o >>= 1) {
      KSum b{__shfl_down_sync(0xffffffffu, acc.s, o),
             __shfl_down_sync(0xffffffffu, acc.c, o)};
      acc = merge(acc, b);
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
  }
}

double device_sum(const double* d, uint64_t n, cudaStream_t s) {
  const int blocks = 148 * 4, threads = 256;
  DevBuf<KSum> part(blocks);
  k_sum<<<blocks, threads, 0, s>>>(d, n, part.get());
  LBM_CHECK_LAUNCH();
  std::vector<KSum> h(blocks);
  LBM_CUDA(cudaMemcpyAsync(h.data(), part.get(), blocks * sizeof(KSum),
                           cudaMemcpyDeviceToHost, s));
  LBM_CUDA(cudaStreamSynchronize(s));
  double sum = 0.0, c = 0.0;
  for (const KSum& k : h) {
    for (double v : {k.s, k.c}) {
      const double t = sum + v;
      if (std::fabs(sum) >= std::fabs(v))
        c += (sum - t) + v;
      else
        c += (v - t) + sum;
      sum = t;
    }
  }
  return sum + c;
}

// ---- per-kernel event statistics --------------------------------------------
cudaEvent_t KernelStats::get_event() {
  if (!pool_.empty()) {
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  LBM_CUDA(cudaEventCreate(&e));
  return e;
}

int occupancy_blocks(const void* kern, int threads) {
  static std::mutex m;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lk(m);
  auto it = cache.find({kern, threads});
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  LBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0));
  cache[{kern, threads}] = per_sm;
  return per_sm;
}

int KernelStats::begin(const char* name, cudaStream_t s, long sweeps) {
  ++launches_;
  if (!on_) return -1;
  int row = -1;
  for (size_t i = 0; i < rows_.size(); ++i)
    if (rows_[i].name == name) row = static_cast<int>(i);
  if (row < 0) {
    rows_.push_back({name, 0, 0.0});
    row = static_cast<int>(rows_.size()) - 1;
  }
  Pending p{row, get_event(), get_event(), sweeps};
  LBM_CUDA(cudaEventRecord(p.a, s));
  if (!origin_) {
    origin_ = get_event();
    LBM_CUDA(cudaEventRecord(origin_, s));
  }
  pending_.push_back(p);
  return static_cast<int>(pending_.size()) - 1;
}

void KernelStats::end(int token, cudaStream_t s) {
  if (token < 0) return;
  LBM_CUDA(cudaEventRecord(pending_[token].b, s));
}

void KernelStats::collect() {
  for (Pending& p : pending_) {
    LBM_CUDA(cudaEventSynchronize(p.b));
    float ms = 0.f;
    LBM_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    rows_[p.row].launches += p.sweeps;
    rows_[p.row].ms += ms;
    if (origin_ && spans_.size() < kMaxSpans) {
      float t0 = 0.f, t1 = 0.f;
      LBM_CUDA(cudaEventElapsedTime(&t0, origin_, p.a));
      LBM_CUDA(cudaEventElapsedTime(&t1, origin_, p.b));
      spans_.push_back({p.row, t0, t1});
    }
    pool_.push_back(p.a);
    pool_.push_back(p.b);
  }
  pending_.clear();
}

void KernelStats::reset() {
  collect();
  rows_.clear();
  spans_.clear();
  if (origin_) pool_.push_back(origin_);
  origin_ = nullptr;
}

KernelStats::~KernelStats() {
  for (Pending& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (cudaEvent_t e : pool_) cudaEventDestroy(e);
  if (origin_) cudaEventDestroy(origin_);
}

}  // namespace lbmgpu

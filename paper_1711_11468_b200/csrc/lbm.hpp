// Internal C++ interface of the B200 LBM sweep library (behind include/lbmgpu.h).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <nvtx3/nvToolsExtCudaRt.h>

#include "common.cuh"
#include "model.cuh"

namespace lbmgpu {

// ---------------------------------------------------------------- registry
enum class Prop { OsPush = 0, OsPull = 1, Aa = 2 };

// lbm::KernelDescriptor (reference include/lbm/kernels.hpp:25-36)
struct Descriptor {
  std::string name;
  Prop prop = Prop::OsPush;
  bool soa = true;
  bool indirect = false;
  int blk = 0;
  int nt_streams = 0;
  bool ria = false, pv = false, vec = false;
  int vector_width = 4;
};

const std::vector<std::string>& kernel_names();
Descriptor make_descriptor(const std::string& name, int blk, int vector_width);

struct LoopBalance {
  double ref_min = 0, ref_max = 0;  // reference B_l incl. CPU write-allocate
  double gpu = 0;                   // algorithmic bytes per FLUP on the GPU
};
// geometry statistics (RIA names): total_runs < 0 = none
LoopBalance loop_balance(const Descriptor& d, int64_t total_runs = -1, int64_t n_fluid = 0);
struct Roofline {
  double pmax_min_mflups = 0, pmax_max_mflups = 0;
};
Roofline roofline(double gbps, double bl_min, double bl_max);

// --------------------------------------------------------------- geometry
enum GeomKind { kChannel = 0, kSlit = 1, kPipe = 2, kBlocks = 3, kCustom = 4 };

struct GeomSpec {
  int kind = kChannel;
  int nx = 500, ny = 100, nz = 100;
  int block = 4, spacing = 4;
  int pipe_diameter = 0;
  std::vector<uint8_t> custom;  // kCustom: canonical flags
  bool custom_periodic[3] = {false, false, false};
  uint64_t volume() const { return uint64_t(nx) * ny * nz; }
};

// Reference build_geometry's argument checks (geometry.cpp:17-25,48-104),
// raised before any allocation; returns the per-axis periodicity.
std::array<bool, 3> validate_geometry(const GeomSpec& g);

// ----------------------------------------------------------------- padding
struct Padding {
  int mode = 1;  // 0 none, 1 auto, 2 thrash, 3 explicit
  std::array<int64_t, kQ> pads{};
};
std::array<uint64_t, kQ> padding_offsets(uint64_t n_fluid, const Padding& p,
                                         uint64_t* total);

// ------------------------------------------------------- device buffers
// Guard zones (debug aid, LBMGPU_GUARD=1 at allocation time; the pool has no
// compute-sanitizer): every device buffer gets kGuardBytes of a known byte
// pattern on both sides, and guard_check() reports buffers whose guards a
// kernel overwrote.  Off by default (plain cudaMalloc).
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_enabled();
void* guarded_malloc(size_t bytes);   // returns the user pointer
void guarded_free(void* user);
int guard_check(std::string* report);  // number of corrupted buffers
int guard_selftest();                  // negative control: 1 expected

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), guarded_(o.guarded_) {
    o.p_ = nullptr;
    o.n_ = 0;
    o.guarded_ = false;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      guarded_ = o.guarded_;
      o.p_ = nullptr;
      o.n_ = 0;
      o.guarded_ = false;
    }
    return *this;
  }
  void alloc(size_t n) {
    release();
    if (n) {
      if (guard_enabled()) {
        p_ = static_cast<T*>(guarded_malloc(n * sizeof(T)));
        guarded_ = true;
      } else {
        LBM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
      }
    }
    n_ = n;
  }
  void release() {
    if (p_) {
      if (guarded_)
        guarded_free(p_);
      else
        cudaFree(p_);
    }
    p_ = nullptr;
    n_ = 0;
    guarded_ = false;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }
  // byte offset of get() inside its cudaMalloc allocation (CUDA IPC handles
  // name the allocation base)
  size_t alloc_offset() const { return guarded_ ? kGuardBytes : 0; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  bool guarded_ = false;
};

// Device-resident FlagField (geometry.hpp:16-29): canonical x-major order.
struct DeviceGeometry {
  int nx = 0, ny = 0, nz = 0;
  std::array<bool, 3> periodic{};
  DevBuf<uint8_t> flags;  // V bytes, 1 = solid
  int64_t n_fluid = 0;
  uint64_t volume() const { return uint64_t(nx) * ny * nz; }
};
DeviceGeometry build_geometry_device(const GeomSpec& g, cudaStream_t s);

// Exclusive prefix count of fluid nodes (flag == 0) over `n` flags; returns
// the total.  out may alias nothing; n < 2^32.
uint64_t scan_fluid(const uint8_t* flags, uint32_t* out, uint64_t n,
                    cudaStream_t s);

// ------------------------------------------------------------ statistics
class KernelStats {
 public:
  void enable(bool on) { on_ = on; }
  bool enabled() const { return on_; }
  // Records a (start) event before a launch; returns a token for end().
  // `sweeps` = lattice sweeps the launch performs (a fused multi-step launch
  // counts T); the per-row "launches" total is in sweeps.
  int begin(const char* name, cudaStream_t s, long sweeps = 1);
  void end(int token, cudaStream_t s);
  void collect();  // synchronises pending events into the totals
  void reset();
  struct Row { std::string name; long launches = 0; double ms = 0; };
  const std::vector<Row>& rows() { collect(); return rows_; }
  // Per-launch intervals (ms after the first recorded launch of this
  // enable/reset period; events on every stream share the device clock),
  // the evidence that boundary-stream work overlaps the interior sweeps.
  struct Span { int row; double t0, t1; };
  const std::vector<Span>& timeline() { collect(); return spans_; }
  long launches() const { return launches_; }
  void count_launch() { ++launches_; }
  void add_launches(long n) { launches_ += n; }
  ~KernelStats();

 private:
  struct Pending { int row; cudaEvent_t a, b; long sweeps; };
  static constexpr size_t kMaxSpans = 1 << 16;
  std::vector<Span> spans_;
  cudaEvent_t origin_ = nullptr;  // first event of the period (a Pending's start)
  bool on_ = false;
  long launches_ = 0;
  std::vector<Row> rows_;
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> pool_;
  cudaEvent_t get_event();
};

// Device micro-benchmarks (microbench.cu): one pass's element count per
// stream and accounted bytes (GPU: no write allocate; ref: the reference's
// CPU accounting, microbench.cpp:92-99).
struct MicroPlan {
  int streams = 1, arrays = 2;
  uint64_t n = 0, bytes_gpu = 0, bytes_ref = 0;
};
MicroPlan micro_plan(const std::string& kind, uint64_t working_set_bytes);

// NVTX range over a host scope (header-only NVTX 3: a no-op unless a tool
// such as nsys is attached).  The engines mark each advance() and, on the
// decomposed paths, each sub-step's boundary / interior enqueue; their two
// streams are named "lbmgpu interior" / "lbmgpu boundary".
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Resident blocks per SM of a kernel at a block size (no dynamic shared
// memory), cached: the fused launches query it on every advance().
int occupancy_blocks(const void* kern, int threads);

// ------------------------------------------------------------- engines
// Distribution request (see lbmgpu_dist in include/lbmgpu.h).
struct DistSpec {
  int rank = 0, nranks = 1, device = -1, virtual_parts = 1;
  std::array<uint8_t, 128> nccl_id{};
  bool have_id = false;
  int transport = 0;  // 0: halo copies (NCCL / device), 1: peer memory (direct z slabs)
};

// One GPU-resident sweep implementation of the reference's Kernel
// (include/lbm/kernels.hpp:58-96).  All calls come from one host thread.
class Engine {
 public:
  virtual ~Engine() = default;
  const Descriptor& descriptor() const { return desc_; }
  uint64_t n_fluid() const { return n_fluid_; }
  cudaStream_t stream() const { return stream_; }
  KernelStats& stats() { return stats_; }

  // steps already validated (>= 0, even for AA).
  virtual void advance(const TrtArgs& t, long steps) = 0;

  // Throws if the engine's stream work failed in a way only the device can
  // see (peer transport: a neighbour's signal timed out).  Synchronises.
  virtual void check_health() {}

  // Canonical nodes [c0, c0+count) -> device staging (count*19 doubles,
  // node-major) and back.  Runs on stream().
  virtual void gather_canonical(uint64_t c0, uint64_t count, double* d_out) = 0;
  virtual void scatter_canonical(uint64_t c0, uint64_t count,
                                 const double* d_in) = 0;
  // Perturbed equilibrium generated per canonical index (harness.cpp:50-62).
  virtual void load_perturbed(uint64_t seed, double amplitude) = 0;
  virtual double total_mass() = 0;
  // Device macro fields over canonical nodes: rho (N) and u (3N); the engine
  // owns the arrays.  Returns device pointers.
  virtual void macro_fields(double* d_rho, double* d_u) = 0;

  // Pipelined job: load_state(host_in) + advance(steps) + snapshot(host_out)
  // with the host transfers overlapped with the sweeps (pinned host buffers
  // of n_fluid * 19 doubles).  Returns false, having done nothing, when the
  // engine cannot pipeline this job; the caller then runs the plain
  // sequence.  Bitwise the plain sequence's result.
  virtual bool run_job(const TrtArgs& t, long steps, const double* host_in, double* host_out) {
    (void)t; (void)steps; (void)host_in; (void)host_out;
    return false;
  }

  // list structure export (ConfigError for direct engines)
  virtual void export_structure(int32_t* nodes, uint32_t* adj,
                                uint64_t* starts, uint64_t* total) {
    (void)nodes; (void)adj; (void)starts; (void)total;
    throw ConfigError("kernel '" + desc_.name +
                      "' uses direct addressing and has no list structure");
  }
  virtual bool ria_stats(int64_t* runs, double* vfrac) {
    (void)runs; (void)vfrac;
    return false;
  }
  // run-coded names: vectorizable_fraction at any width, the run starts
  virtual bool ria_vector_fraction(int w, double* v) {
    (void)w; (void)v;
    return false;
  }
  virtual bool ria_run_starts(std::vector<uint32_t>& out) {
    (void)out;
    return false;
  }
  // Peer-memory transport (nranks > 1): this rank's CUDA IPC record, and
  // the attach of every rank's record (rank order).
  virtual void peer_export(std::vector<uint8_t>& rec) {
    (void)rec;
    throw ConfigError("peer transport: not enabled for this lattice");
  }
  virtual void peer_attach(const uint8_t* recs, size_t rec_len, int nranks) {
    (void)recs; (void)rec_len; (void)nranks;
    throw ConfigError("peer transport: not enabled for this lattice");
  }
  virtual void peer_probe(int which, std::vector<double>& out) {
    (void)which; (void)out;
    throw ConfigError("peer transport: not enabled for this lattice");
  }
  virtual int parts() const { return 1; }
  virtual void part_info(int p, int* z0, int* z1, uint64_t* nf) const {
    (void)p; *z0 = 0; *z1 = 0; *nf = n_fluid_;
  }
  // Whether this process holds every canonical node (false when the domain
  // is split across processes).
  virtual bool holds_all() const { return true; }
  // Process-local rows: this process's fluid nodes in canonical order.
  virtual uint64_t local_rows() const { return n_fluid_; }
  virtual void local_canonical_index(uint64_t* out) const {
    for (uint64_t k = 0; k < n_fluid_; ++k) out[k] = k;
  }
  // Local rows [k0, k0+count) <-> device staging (count*19, node-major).
  virtual void gather_local(uint64_t k0, uint64_t count, double* d,
                            bool to_staging) {
    if (to_staging)
      gather_canonical(k0, count, d);
    else
      scatter_canonical(k0, count, d);
  }

 protected:
  Descriptor desc_;
  uint64_t n_fluid_ = 0;
  cudaStream_t stream_ = nullptr;
  KernelStats stats_;
};

std::unique_ptr<Engine> make_direct_engine(const Descriptor& d,
                                           const GeomSpec& g,
                                           const DistSpec& dist);
std::unique_ptr<Engine> make_list_engine(const Descriptor& d,
                                         const GeomSpec& g,
                                         const Padding& pad,
                                         const DistSpec& dist);

// ---------------------------------------------------- device primitives
// Kahan/Neumaier-compensated sum of n doubles accessed through idx.
double device_sum(const double* d, uint64_t n, cudaStream_t s);

// splitmix64 (harness.cpp:18-23)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// perturbed_equilibrium value for (canonical n, d) (harness.cpp:50-62)
__host__ __device__ __forceinline__ double perturbed_value(uint64_t n, int d,
                                                           uint64_t seed,
                                                           double amplitude) {
  const uint64_t h = splitmix64(seed ^ (n * kQ + static_cast<uint64_t>(d)));
  const double u01 = static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0);
  return weight(d) * (1.0 + amplitude * (u01 - 0.5));
}

}  // namespace lbmgpu

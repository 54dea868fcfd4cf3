// extern "C" boundary (include/lbmgpu.h) over the device engines.
#include "../../include/lbmgpu.h"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "halo.hpp"
#include "lbm.hpp"

using namespace lbmgpu;

struct lbmgpu_ctx {
  std::unique_ptr<Engine> eng;
  Descriptor desc;
  GeomSpec geom;
  DevBuf<double> rho, u, uprev;  // steady-state scratch
  cudaStream_t copy = nullptr;   // host<->device staging copies
  // staging buffers and events of pipelined(), kept across calls (a
  // load/snapshot of a small lattice would otherwise pay for the
  // allocations more than for the transfer)
  DevBuf<double> stage[2];
  cudaEvent_t ready[2] = {}, freed[2] = {};
  ~lbmgpu_ctx() {
    for (int b = 0; b < 2; ++b) {
      if (ready[b]) cudaEventDestroy(ready[b]);
      if (freed[b]) cudaEventDestroy(freed[b]);
    }
    if (copy) cudaStreamDestroy(copy);
  }
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return LBMGPU_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return LBMGPU_ECONFIG;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return LBMGPU_ENUMERICAL;
  } catch (const DeviceError& e) {
    g_err = e.what();
    return LBMGPU_EDEVICE;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return LBMGPU_EDEVICE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LBMGPU_EDEVICE;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw ConfigError(std::string(what) + " must not be NULL");
}

GeomSpec to_spec(const lbmgpu_geometry* g) {
  need(g, "geometry");
  GeomSpec s;
  s.kind = g->kind;
  s.nx = g->nx;
  s.ny = g->ny;
  s.nz = g->nz;
  s.block = g->block;
  s.spacing = g->spacing;
  s.pipe_diameter = g->pipe_diameter;
  if (g->kind == kCustom) {
    need(g->flags, "custom geometry flags");
    if (g->nx < 1 || g->ny < 1 || g->nz < 1)
      throw ConfigError("custom geometry: dims must be >= 1");
    s.custom.assign(g->flags, g->flags + s.volume());
    for (int a = 0; a < 3; ++a) s.custom_periodic[a] = g->periodic[a] != 0;
  }
  return s;
}

Padding to_padding(const lbmgpu_padding* p) {
  Padding q;
  if (p) {
    q.mode = p->mode;
    for (int d = 0; d < kQ; ++d) q.pads[d] = p->pads[d];
  }
  return q;
}

void fill_desc(const Descriptor& d, lbmgpu_descriptor* o) {
  o->prop = static_cast<int>(d.prop);
  o->layout_soa = d.soa;
  o->indirect = d.indirect;
  o->blk = d.blk;
  o->nt_streams = d.nt_streams;
  o->ria = d.ria;
  o->pv = d.pv;
  o->vec = d.vec;
  o->vector_width = d.vector_width;
}

// TrtParams::validate (d3q19.hpp:75-81) + Kernel::advance checks
// (kernels.cpp:84-93).
TrtArgs checked_trt(lbmgpu_ctx* c, double wp, double lambda, const double* g,
                    long steps) {
  if (steps < 0) throw ConfigError("advance: steps must be >= 0");
  if (!(wp > 0.0) || !(wp < 2.0))
    throw ConfigError("TrtParams: omega_plus must be in (0, 2), got " +
                      std::to_string(wp));
  if (!(lambda > 0.0)) throw ConfigError("TrtParams: magic_lambda must be positive");
  if (c->desc.prop == Prop::Aa && steps % 2 != 0)
    throw ConfigError("kernel '" + c->desc.name +
                      "' uses the AA pattern and requires an even step count, "
                      "got " + std::to_string(steps));
  need(g, "g");
  return make_trt(wp, omega_minus_of(wp, lambda), g);
}

constexpr uint64_t kChunkNodes = 1ull << 21;  // 2 Mi nodes = 304 MiB staging

struct HostPinned {
  void* p = nullptr;
  explicit HostPinned(size_t b) { LBM_CUDA(cudaMallocHost(&p, b)); }
  ~HostPinned() {
    if (p) cudaFreeHost(p);
  }
};

// Host <-> device transfer of `rows` node rows (19 doubles each) through two
// staging buffers: the layout conversion (dev: gather/scatter kernel) runs on
// the engine stream, the PCIe copies on a copy stream, so chunk k's copy
// overlaps chunk k+1's kernel.  dev(row0, n, staging, to_host).
template <class Dev>
void pipelined(lbmgpu_ctx* c, double* host, uint64_t rows, bool to_host, Dev dev) {
  if (rows == 0) return;
  if (!c->copy) LBM_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  const uint64_t chunk = std::min(rows, kChunkNodes);
  const int nb = rows > chunk ? 2 : 1;
  for (int b = 0; b < nb; ++b) {
    if (c->stage[b].size() < chunk * kQ) c->stage[b].alloc(chunk * kQ);
    if (!c->ready[b]) LBM_CUDA(cudaEventCreateWithFlags(&c->ready[b], cudaEventDisableTiming));
    if (!c->freed[b]) LBM_CUDA(cudaEventCreateWithFlags(&c->freed[b], cudaEventDisableTiming));
  }
  cudaStream_t s = c->eng->stream(), cs = c->copy;
  cudaEvent_t* ready = c->ready;
  cudaEvent_t* freed = c->freed;
  try {
    uint64_t k = 0;
    for (uint64_t r0 = 0; r0 < rows; r0 += chunk, ++k) {
      const int b = static_cast<int>(k & 1);
      const uint64_t n = std::min(chunk, rows - r0);
      double* sb = c->stage[b].get();
      if (to_host) {
        if (k >= 2) LBM_CUDA(cudaStreamWaitEvent(s, freed[b], 0));
        dev(r0, n, sb, true);
        LBM_CUDA(cudaEventRecord(ready[b], s));
        LBM_CUDA(cudaStreamWaitEvent(cs, ready[b], 0));
        LBM_CUDA(cudaMemcpyAsync(host + r0 * kQ, sb, n * kQ * 8, cudaMemcpyDeviceToHost, cs));
        LBM_CUDA(cudaEventRecord(freed[b], cs));
      } else {
        // (every call ends with both streams synchronised, so a buffer's
        // first use in a call needs no wait)
        if (k >= 2) LBM_CUDA(cudaStreamWaitEvent(cs, freed[b], 0));
        LBM_CUDA(cudaMemcpyAsync(sb, host + r0 * kQ, n * kQ * 8, cudaMemcpyHostToDevice, cs));
        LBM_CUDA(cudaEventRecord(ready[b], cs));
        LBM_CUDA(cudaStreamWaitEvent(s, ready[b], 0));
        dev(r0, n, sb, false);
        LBM_CUDA(cudaEventRecord(freed[b], s));
      }
    }
    LBM_CUDA(cudaStreamSynchronize(cs));
    LBM_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(s);
    throw;
  }
}

uint64_t fnv_bytes(uint64_t h, const unsigned char* p, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// equilibrium(rho, u) (reference src/d3q19.cpp:7-18)
void equilibrium(double rho, const double* u, double* f) {
  if (!(rho > 0.0))
    throw ConfigError("equilibrium: rho must be positive, got " + std::to_string(rho));
  const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int i = 0; i < kQ; ++i) {
    const double cu = static_cast<double>(cx(i)) * u[0] +
                      static_cast<double>(cy(i)) * u[1] +
                      static_cast<double>(cz(i)) * u[2];
    f[i] = weight(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
  }
}

}  // namespace

// device helpers implemented in harness.cu
namespace lbmgpu {
void velocity_change(const double* u, const double* uprev, uint64_t n3,
                     double* max_du, double* max_u, bool* finite,
                     cudaStream_t s);
void layer_sums(const double* u, uint64_t cols, int layers, double* out_dev,
                cudaStream_t s);
double run_microbench(const std::string& kind, uint64_t working_set_bytes, int reps);
}  // namespace lbmgpu

extern "C" {

const char* lbmgpu_last_error(void) { return g_err.c_str(); }

uint64_t lbmgpu_fnv1a(const void* data, uint64_t nbytes) {
  return fnv_bytes(0xcbf29ce484222325ull, static_cast<const unsigned char*>(data),
                   nbytes);
}
int lbmgpu_abi_version(void) { return LBMGPU_ABI_VERSION; }

int lbmgpu_guard_check(int* corrupted) {
  return guard([&] {
    need(corrupted, "corrupted");
    std::string rep;
    *corrupted = guard_check(&rep);
    if (*corrupted) g_err = "guard zones overwritten: " + rep;
  });
}

int lbmgpu_guard_selftest(int* detected) {
  return guard([&] {
    need(detected, "detected");
    *detected = guard_selftest();
  });
}

int lbmgpu_kernel_names(char* buf, size_t cap) {
  return guard([&] {
    std::string s;
    for (const auto& n : kernel_names()) s += n + "\n";
    if (!buf || s.size() + 1 > cap) throw ConfigError("kernel_names: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int lbmgpu_make_descriptor(const char* name, int blk, int W,
                           lbmgpu_descriptor* out) {
  return guard([&] {
    need(name, "name");
    need(out, "out");
    fill_desc(make_descriptor(name, blk, W), out);
  });
}

int lbmgpu_padding_offsets(uint64_t n, const lbmgpu_padding* pad,
                           uint64_t* starts, uint64_t* total) {
  return guard([&] {
    need(starts, "starts");
    uint64_t t = 0;
    auto s = padding_offsets(n, to_padding(pad), &t);
    for (int d = 0; d < kQ; ++d) starts[d] = s[d];
    if (total) *total = t;
  });
}

int lbmgpu_loop_balance(const char* name, double* a, double* b, double* g) {
  return guard([&] {
    need(name, "name");
    LoopBalance l = loop_balance(make_descriptor(name, 0, 4));
    if (a) *a = l.ref_min;
    if (b) *b = l.ref_max;
    if (g) *g = l.gpu;
  });
}

int lbmgpu_loop_balance_stats(const char* name, int64_t total_runs, int64_t n_fluid, double* a,
                              double* b, double* g) {
  return guard([&] {
    need(name, "name");
    LoopBalance l = loop_balance(make_descriptor(name, 0, 4), total_runs, n_fluid);
    if (a) *a = l.ref_min;
    if (b) *b = l.ref_max;
    if (g) *g = l.gpu;
  });
}

int lbmgpu_roofline(double gbps, double bl_min, double bl_max, double* pmax_min, double* pmax_max) {
  return guard([&] {
    Roofline r = roofline(gbps, bl_min, bl_max);
    if (pmax_min) *pmax_min = r.pmax_min_mflups;
    if (pmax_max) *pmax_max = r.pmax_max_mflups;
  });
}

double lbmgpu_omega_minus(double wp, double lambda) {
  return omega_minus_of(wp, lambda);
}

int lbmgpu_geometry_build(const lbmgpu_geometry* g, uint8_t* flags_out,
                          int64_t* n_fluid, int* periodic_out) {
  return guard([&] {
    GeomSpec s = to_spec(g);
    validate_geometry(s);  // ConfigError before any device work
    cudaStream_t st;
    LBM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      DeviceGeometry dg = build_geometry_device(s, st);
      if (flags_out)
        LBM_CUDA(cudaMemcpyAsync(flags_out, dg.flags.get(), dg.volume(),
                                 cudaMemcpyDeviceToHost, st));
      LBM_CUDA(cudaStreamSynchronize(st));
      if (n_fluid) *n_fluid = dg.n_fluid;
      if (periodic_out)
        for (int a = 0; a < 3; ++a) periodic_out[a] = dg.periodic[a];
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
  });
}

int lbmgpu_create(const char* name, int blk, int W, const lbmgpu_geometry* geom,
                  const lbmgpu_padding* pad, int row_pad,
                  const lbmgpu_dist* dist, lbmgpu_ctx** out) {
  return guard([&] {
    need(name, "kernel name");
    need(out, "out");
    *out = nullptr;
    if (row_pad < 0) throw ConfigError("FullLattice: row_pad must be >= 0");
    auto c = std::make_unique<lbmgpu_ctx>();
    c->desc = make_descriptor(name, blk, W);
    c->geom = to_spec(geom);
    validate_geometry(c->geom);  // ConfigError before any allocation
    DistSpec ds;
    if (dist) {
      ds.rank = dist->rank;
      ds.nranks = dist->nranks;
      ds.device = dist->device;
      ds.virtual_parts = dist->virtual_parts;
      ds.transport = dist->transport;
      if (dist->nccl_id) {
        std::memcpy(ds.nccl_id.data(), dist->nccl_id, 128);
        ds.have_id = true;
      }
      if (ds.nranks < 1 || ds.rank < 0 || ds.rank >= ds.nranks)
        throw ConfigError("dist: bad rank/nranks");
      if (ds.virtual_parts > 1 && ds.nranks > 1)
        throw ConfigError("dist: virtual_parts needs nranks == 1");
    }
    if (ds.device >= 0) LBM_CUDA(cudaSetDevice(ds.device));
    if (c->desc.indirect) {
      if (ds.transport == 1)
        throw ConfigError("peer transport: implemented for the direct SoA z slabs (kernel '" +
                          c->desc.name + "')");
      if ((ds.nranks > 1 || ds.virtual_parts > 1) &&
          (c->desc.prop != Prop::Aa || c->desc.ria || c->desc.blk != 0))
        throw ConfigError("list decomposition is implemented for list-aa-soa / list-aa-aos "
                          "with blk = 0 (kernel '" + c->desc.name + "')");
      c->eng = make_list_engine(c->desc, c->geom, to_padding(pad), ds);
    } else {
      c->eng = make_direct_engine(c->desc, c->geom, ds);
    }
    *out = c.release();
  });
}

int lbmgpu_destroy(lbmgpu_ctx* c) {
  return guard([&] { delete c; });
}

int lbmgpu_advance(lbmgpu_ctx* c, double wp, double lambda, const double* g,
                   long steps) {
  return guard([&] {
    need(c, "ctx");
    TrtArgs t = checked_trt(c, wp, lambda, g, steps);
    if (steps == 0) return;
    c->eng->advance(t, steps);
    LBM_CUDA(cudaStreamSynchronize(c->eng->stream()));
    c->eng->check_health();
  });
}

int lbmgpu_time_advance(lbmgpu_ctx* c, double wp, double lambda,
                        const double* g, long steps, double* ms) {
  return guard([&] {
    need(c, "ctx");
    need(ms, "ms");
    TrtArgs t = checked_trt(c, wp, lambda, g, steps);
    cudaEvent_t a, b;
    LBM_CUDA(cudaEventCreate(&a));
    LBM_CUDA(cudaEventCreate(&b));
    LBM_CUDA(cudaEventRecord(a, c->eng->stream()));
    if (steps) c->eng->advance(t, steps);
    LBM_CUDA(cudaEventRecord(b, c->eng->stream()));
    LBM_CUDA(cudaEventSynchronize(b));
    float f = 0.f;
    LBM_CUDA(cudaEventElapsedTime(&f, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    c->eng->check_health();
    *ms = f;
  });
}

int lbmgpu_n_fluid(lbmgpu_ctx* c, uint64_t* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    *out = c->eng->n_fluid();
  });
}

int lbmgpu_snapshot(lbmgpu_ctx* c, double* host, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    const uint64_t N = c->eng->n_fluid();
    if (count != N * kQ)
      throw ConfigError("snapshot: buffer holds " + std::to_string(count) +
                        " values, lattice has " + std::to_string(N * kQ));
    need(host, "host buffer");
    c->eng->check_health();
    pipelined(c, host, N, true, [&](uint64_t c0, uint64_t n, double* st, bool) {
      c->eng->gather_canonical(c0, n, st);
    });
  });
}

int lbmgpu_load_state(lbmgpu_ctx* c, const double* host, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    const uint64_t N = c->eng->n_fluid();
    if (count != N * kQ)
      throw ConfigError("load_state: state size does not match fluid count");
    need(host, "host buffer");
    pipelined(c, const_cast<double*>(host), N, false,
              [&](uint64_t c0, uint64_t n, double* st, bool) {
                c->eng->scatter_canonical(c0, n, st);
              });
  });
}

// page-locked (cudaHostAlloc / registered) over [p, p + bytes)
static bool pinned_range(const void* p, size_t bytes) {
  for (const char* q : {static_cast<const char*>(p), static_cast<const char*>(p) + bytes - 1}) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

int lbmgpu_run(lbmgpu_ctx* c, double wp, double lambda, const double* g, long steps,
               const double* host_in, uint64_t in_count, double* host_out, uint64_t out_count,
               int* pipelined_out) {
  return guard([&] {
    need(c, "ctx");
    const uint64_t N = c->eng->n_fluid();
    if (in_count != N * kQ)
      throw ConfigError("load_state: state size does not match fluid count");
    need(host_in, "host buffer");
    TrtArgs t = checked_trt(c, wp, lambda, g, steps);
    if (out_count != N * kQ)
      throw ConfigError("snapshot: buffer holds " + std::to_string(out_count) +
                        " values, lattice has " + std::to_string(N * kQ));
    need(host_out, "host buffer");
    if (pipelined_out) *pipelined_out = 0;
    bool done = false;
    if (c->eng->holds_all() && N && pinned_range(host_in, N * kQ * 8) &&
        pinned_range(host_out, N * kQ * 8)) {
      c->eng->check_health();
      done = c->eng->run_job(t, steps, host_in, host_out);
      if (done) c->eng->check_health();
    }
    if (done) {
      if (pipelined_out) *pipelined_out = 1;
      return;
    }
    int rc = lbmgpu_load_state(c, host_in, in_count);
    if (rc == LBMGPU_OK) rc = lbmgpu_advance(c, wp, lambda, g, steps);
    if (rc == LBMGPU_OK) rc = lbmgpu_snapshot(c, host_out, out_count);
    if (rc != LBMGPU_OK) {
      const std::string m = g_err;
      if (rc == LBMGPU_ECONFIG) throw ConfigError(m);
      if (rc == LBMGPU_ENUMERICAL) throw NumericalError(m);
      throw DeviceError(m);
    }
  });
}

int lbmgpu_local_rows(lbmgpu_ctx* c, uint64_t* rows) {
  return guard([&] {
    need(c, "ctx");
    need(rows, "rows");
    *rows = c->eng->local_rows();
  });
}

int lbmgpu_local_canonical_index(lbmgpu_ctx* c, uint64_t* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    c->eng->local_canonical_index(out);
  });
}

static void local_transfer(lbmgpu_ctx* c, double* host, uint64_t count,
                           bool to_host) {
  const uint64_t R = c->eng->local_rows();
  if (count != R * kQ)
    throw ConfigError("local state: buffer holds " + std::to_string(count) +
                      " values, this process has " + std::to_string(R * kQ));
  need(host, "host buffer");
  pipelined(c, host, R, to_host, [&](uint64_t k0, uint64_t n, double* st, bool th) {
    c->eng->gather_local(k0, n, st, th);
  });
}

int lbmgpu_snapshot_local(lbmgpu_ctx* c, double* host, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    c->eng->check_health();
    local_transfer(c, host, count, true);
  });
}

int lbmgpu_load_state_local(lbmgpu_ctx* c, const double* host, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    local_transfer(c, const_cast<double*>(host), count, false);
  });
}

int lbmgpu_load_perturbed(lbmgpu_ctx* c, uint64_t seed, double amplitude) {
  return guard([&] {
    need(c, "ctx");
    c->eng->load_perturbed(seed, amplitude);
    LBM_CUDA(cudaStreamSynchronize(c->eng->stream()));
  });
}

int lbmgpu_total_mass(lbmgpu_ctx* c, double* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    c->eng->check_health();
    *out = c->eng->total_mass();
  });
}

int lbmgpu_fingerprint(lbmgpu_ctx* c, uint64_t* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    if (!c->eng->holds_all())
      throw ConfigError("fingerprint: the state is split across processes; "
                        "gather the local rows (lbmgpu_snapshot_local) first");
    c->eng->check_health();
    const uint64_t N = c->eng->n_fluid();
    const uint64_t chunk = std::min(N, kChunkNodes);
    cudaStream_t s = c->eng->stream();
    DevBuf<double> stage[2] = {DevBuf<double>(chunk * kQ), DevBuf<double>(chunk * kQ)};
    HostPinned pin0(chunk * kQ * 8), pin1(chunk * kQ * 8);
    void* pins[2] = {pin0.p, pin1.p};
    cudaEvent_t ev[2];
    LBM_CUDA(cudaEventCreate(&ev[0]));
    LBM_CUDA(cudaEventCreate(&ev[1]));
    uint64_t h = 0xcbf29ce484222325ull;
    const uint64_t nchunks = ceil_div(N, chunk);
    auto issue = [&](uint64_t k) {
      const uint64_t c0 = k * chunk, n = std::min(chunk, N - c0);
      const int b = static_cast<int>(k & 1);
      c->eng->gather_canonical(c0, n, stage[b].get());
      LBM_CUDA(cudaMemcpyAsync(pins[b], stage[b].get(), n * kQ * 8,
                               cudaMemcpyDeviceToHost, s));
      LBM_CUDA(cudaEventRecord(ev[b], s));
    };
    if (nchunks) issue(0);
    for (uint64_t k = 0; k < nchunks; ++k) {
      if (k + 1 < nchunks) issue(k + 1);
      const int b = static_cast<int>(k & 1);
      LBM_CUDA(cudaEventSynchronize(ev[b]));
      const uint64_t n = std::min(chunk, N - k * chunk);
      h = fnv_bytes(h, static_cast<const unsigned char*>(pins[b]), n * kQ * 8);
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    *out = h;
  });
}

int lbmgpu_capabilities(lbmgpu_ctx* c, int* nt_avail, int* nt_eff, int* huge) {
  return guard([&] {
    need(c, "ctx");
    // GPU stores are full-sector writes with no write allocate; the nt names
    // use st.global.cs (evict-first) streaming stores.
    const int nt = c->desc.nt_streams;
    if (nt_avail) *nt_avail = nt > 0 ? 1 : 0;
    if (nt_eff) *nt_eff = nt;
    if (huge) *huge = 0;
  });
}

int lbmgpu_ria_stats(lbmgpu_ctx* c, int64_t* runs, int64_t* nf, double* vfrac,
                     double* pvfrac) {
  return guard([&] {
    need(c, "ctx");
    int64_t r = -1;
    double v = -1.0;
    const bool have = c->eng->ria_stats(&r, &v);
    if (runs) *runs = have ? r : -1;
    if (nf) *nf = have ? static_cast<int64_t>(c->eng->n_fluid()) : -1;
    if (vfrac) *vfrac = have ? v : -1.0;
    if (pvfrac) *pvfrac = (have && c->desc.pv) ? v : -1.0;
  });
}

int lbmgpu_vectorizable_fraction(lbmgpu_ctx* c, int width, double* v) {
  return guard([&] {
    need(c, "ctx");
    need(v, "out");
    if (!c->eng->ria_vector_fraction(width, v)) *v = -1.0;
  });
}

int lbmgpu_export_runs(lbmgpu_ctx* c, uint32_t* run_starts, uint64_t cap, int64_t* count) {
  return guard([&] {
    need(c, "ctx");
    need(count, "count");
    std::vector<uint32_t> r;
    if (!c->eng->ria_run_starts(r)) {
      *count = -1;
      return;
    }
    *count = static_cast<int64_t>(r.size());
    if (!run_starts) return;
    if (cap < r.size())
      throw ConfigError("export_runs: buffer holds " + std::to_string(cap) + " run starts, coding has " +
                        std::to_string(r.size()));
    std::copy(r.begin(), r.end(), run_starts);
  });
}

int lbmgpu_descriptor_of(lbmgpu_ctx* c, lbmgpu_descriptor* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    fill_desc(c->desc, out);
  });
}

int lbmgpu_export_structure(lbmgpu_ctx* c, int32_t* nodes, uint32_t* adj,
                            uint64_t* starts, uint64_t* total) {
  return guard([&] {
    need(c, "ctx");
    c->eng->export_structure(nodes, adj, starts, total);
  });
}

int lbmgpu_steady_state_run(lbmgpu_ctx* c, double wp, double lambda,
                            const double* g, long interval, double rel_tol,
                            long max_steps, long* steps_out, int* converged,
                            double* final_delta) {
  return guard([&] {
    need(c, "ctx");
    // harness.cpp:141-174
    if (!(rel_tol > 0.0)) throw ConfigError("steady_state_run: rel_tol > 0");
    if (interval < 1) throw ConfigError("steady_state_run: check_interval >= 1");
    if (c->desc.prop == Prop::Aa && interval % 2 != 0) ++interval;
    const uint64_t N = c->eng->n_fluid();
    cudaStream_t s = c->eng->stream();
    if (c->u.size() != 3 * N) {
      c->rho.alloc(N);
      c->u.alloc(3 * N);
      c->uprev.alloc(3 * N);
    }
    c->eng->macro_fields(c->rho.get(), c->uprev.get());
    long steps = 0;
    bool conv = false;
    double delta = 0.0;
    while (steps < max_steps) {
      const long chunk = std::min(interval, max_steps - steps);
      TrtArgs t = checked_trt(c, wp, lambda, g, chunk);
      if (chunk) c->eng->advance(t, chunk);
      steps += chunk;
      c->eng->macro_fields(c->rho.get(), c->u.get());
      double max_du = 0, max_u = 0;
      bool finite = true;
      velocity_change(c->u.get(), c->uprev.get(), 3 * N, &max_du, &max_u,
                      &finite, s);
      if (!finite)
        throw NumericalError("steady_state_run: non-finite velocity at step " +
                             std::to_string(steps));
      delta = max_u > 0.0 ? max_du / max_u : max_du;
      std::swap(c->u, c->uprev);
      if (delta < rel_tol) {
        conv = true;
        break;
      }
    }
    if (steps_out) *steps_out = steps;
    if (converged) *converged = conv;
    if (final_delta) *final_delta = delta;
  });
}

int lbmgpu_layer_ux(lbmgpu_ctx* c, double* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    const GeomSpec& g = c->geom;
    const int layers = g.nz - 2;
    const uint64_t cols = uint64_t(g.nx) * g.ny;
    if (g.kind != kSlit || c->eng->n_fluid() != cols * layers)
      throw ConfigError("layer_ux: needs the slit geometry");
    const uint64_t N = c->eng->n_fluid();
    cudaStream_t s = c->eng->stream();
    DevBuf<double> rho(N), u(3 * N), sums(layers);
    c->eng->macro_fields(rho.get(), u.get());
    layer_sums(u.get(), cols, layers, sums.get(), s);
    LBM_CUDA(cudaMemcpyAsync(out, sums.get(), layers * 8, cudaMemcpyDeviceToHost, s));
    LBM_CUDA(cudaStreamSynchronize(s));
  });
}

int lbmgpu_verify(const char* name, int nx, int ny, int nz, double gx,
                  double tau, double lambda, long interval, double rel_tol,
                  long max_steps, lbmgpu_verify_report* rep, double* simulated,
                  double* analytic) {
  return guard([&] {
    need(name, "kernel name");
    need(rep, "report");
    // PoiseuilleCase::validate (verification.cpp:7-17)
    const double wp = 1.0 / tau;
    if (!(wp > 0.0) || !(wp < 2.0))
      throw ConfigError("TrtParams: omega_plus must be in (0, 2), got " +
                        std::to_string(wp));
    if (!(lambda > 0.0)) throw ConfigError("TrtParams: magic_lambda must be positive");
    if (nz < 6) throw ConfigError("Poiseuille case: nz must be >= 6");
    if (nx < 1 || ny < 1) throw ConfigError("Poiseuille case: bad dims");
    const int layers = nz - 2;
    const double h = layers;
    const double nu = (1.0 / wp - 0.5) / 3.0;  // d3q19.hpp:68
    const double u_max = std::abs(gx) * h * h / (8.0 * nu);
    if (!(u_max < 0.05))
      throw ConfigError("Poiseuille case: centerline velocity g*h^2/(8 nu) = " +
                        std::to_string(u_max) +
                        " is too close to the speed of sound");
    // analytic_profile (verification.cpp:19-29)
    std::vector<double> ana(layers), sim(layers, 0.0);
    for (int k = 0; k < layers; ++k) {
      const double zeta = k + 0.5;
      ana[k] = gx / (2.0 * nu) * zeta * (h - zeta);
    }
    const double shift = gx / 2.0;
    lbmgpu_geometry geo{};
    geo.kind = LBMGPU_SLIT;
    geo.nx = nx;
    geo.ny = ny;
    geo.nz = nz;
    lbmgpu_padding pad{};
    pad.mode = 1;
    lbmgpu_ctx* raw = nullptr;
    int rc = lbmgpu_create(name, 0, 4, &geo, &pad, 0, nullptr, &raw);
    if (rc) {
      if (rc == LBMGPU_ECONFIG) throw ConfigError(g_err);
      throw DeviceError(g_err);
    }
    std::unique_ptr<lbmgpu_ctx> c(raw);
    const uint64_t N = c->eng->n_fluid();
    // warm start (verification.cpp:56-67)
    std::vector<double> state(N * kQ);
    for (uint64_t n = 0; n < N; ++n) {
      const int kz = static_cast<int>(n % layers);
      const double u[3] = {ana[kz] - shift, 0.0, 0.0};
      equilibrium(1.0, u, &state[n * kQ]);
    }
    if ((rc = lbmgpu_load_state(c.get(), state.data(), state.size())))
      throw DeviceError(g_err);
    const double g3[3] = {gx, 0.0, 0.0};
    long steps = 0;
    int conv = 0;
    double delta = 0;
    rc = lbmgpu_steady_state_run(c.get(), wp, lambda, g3, interval, rel_tol,
                                 max_steps, &steps, &conv, &delta);
    if (rc == LBMGPU_ENUMERICAL) throw NumericalError(g_err);
    if (rc == LBMGPU_ECONFIG) throw ConfigError(g_err);
    if (rc) throw DeviceError(g_err);
    std::vector<double> sums(layers);
    if ((rc = lbmgpu_layer_ux(c.get(), sums.data()))) throw DeviceError(g_err);
    const double per_layer = static_cast<double>(uint64_t(nx) * ny);
    for (int k = 0; k < layers; ++k) sim[k] = sums[k] / per_layer + shift;
    double max_ana = 0, max_diff = 0, sa2 = 0, sd2 = 0;
    for (int k = 0; k < layers; ++k) {
      const double d = sim[k] - ana[k];
      max_ana = std::max(max_ana, std::abs(ana[k]));
      max_diff = std::max(max_diff, std::abs(d));
      sa2 += ana[k] * ana[k];
      sd2 += d * d;
    }
    rep->linf_rel = max_ana > 0.0 ? max_diff / max_ana : max_diff;
    rep->l2_rel = sa2 > 0.0 ? std::sqrt(sd2 / sa2) : std::sqrt(sd2);
    rep->half_force_shift = shift;
    rep->steps = steps;
    rep->converged = conv;
    rep->passed = conv && rep->linf_rel < 1e-4;  // kVerifyLinfTolerance
    if (simulated) std::memcpy(simulated, sim.data(), layers * 8);
    if (analytic) std::memcpy(analytic, ana.data(), layers * 8);
  });
}

int lbmgpu_kernel_stats_enable(lbmgpu_ctx* c, int on) {
  return guard([&] {
    need(c, "ctx");
    c->eng->stats().enable(on != 0);
  });
}

int lbmgpu_kernel_stats(lbmgpu_ctx* c, char* names48, long* launches,
                        double* ms, int cap, int* n) {
  return guard([&] {
    need(c, "ctx");
    const auto& rows = c->eng->stats().rows();
    if (n) *n = static_cast<int>(rows.size());
    for (int i = 0; i < cap && i < static_cast<int>(rows.size()); ++i) {
      if (names48) {
        std::strncpy(names48 + 48 * i, rows[i].name.c_str(), 47);
        names48[48 * i + 47] = 0;
      }
      if (launches) launches[i] = rows[i].launches;
      if (ms) ms[i] = rows[i].ms;
    }
  });
}

int lbmgpu_kernel_timeline(lbmgpu_ctx* c, char* names48, double* t0, double* t1, int cap,
                           int* n) {
  return guard([&] {
    need(c, "ctx");
    KernelStats& st = c->eng->stats();
    const auto& spans = st.timeline();
    const auto& rows = st.rows();
    if (n) *n = static_cast<int>(spans.size());
    for (int i = 0; i < cap && i < static_cast<int>(spans.size()); ++i) {
      if (names48) {
        std::strncpy(names48 + 48 * i, rows[spans[i].row].name.c_str(), 47);
        names48[48 * i + 47] = 0;
      }
      if (t0) t0[i] = spans[i].t0;
      if (t1) t1[i] = spans[i].t1;
    }
  });
}

int lbmgpu_kernel_stats_reset(lbmgpu_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    c->eng->stats().reset();
  });
}

int lbmgpu_launch_count(lbmgpu_ctx* c, long* out) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    *out = c->eng->stats().launches();
  });
}

int lbmgpu_host_alloc(size_t bytes, void** out) {
  return guard([&] {
    need(out, "out");
    LBM_CUDA(cudaMallocHost(out, bytes));
  });
}

int lbmgpu_host_free(void* p) {
  return guard([&] { LBM_CUDA(cudaFreeHost(p)); });
}

int lbmgpu_microbench_accounting(const char* kind, uint64_t working_set_bytes,
                                 uint64_t* elems, uint64_t* bytes_gpu, uint64_t* bytes_ref) {
  return guard([&] {
    need(kind, "kind");
    const MicroPlan m = micro_plan(kind, working_set_bytes);
    if (elems) *elems = m.n;
    if (bytes_gpu) *bytes_gpu = m.bytes_gpu;
    if (bytes_ref) *bytes_ref = m.bytes_ref;
  });
}

int lbmgpu_microbench(const char* kind, uint64_t bytes, int reps, double* gbps) {
  return guard([&] {
    need(kind, "kind");
    need(gbps, "gbps");
    *gbps = run_microbench(kind, bytes, reps);
  });
}

int lbmgpu_device_info(int device, char* name64, int* sms, size_t* mem,
                       int* l2) {
  return guard([&] {
    cudaDeviceProp p;
    if (device < 0) LBM_CUDA(cudaGetDevice(&device));
    LBM_CUDA(cudaGetDeviceProperties(&p, device));
    if (name64) {
      std::strncpy(name64, p.name, 63);
      name64[63] = 0;
    }
    if (sms) *sms = p.multiProcessorCount;
    if (mem) *mem = p.totalGlobalMem;
    if (l2) *l2 = p.l2CacheSize;
  });
}

int lbmgpu_synchronize(lbmgpu_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    LBM_CUDA(cudaStreamSynchronize(c->eng->stream()));
  });
}

int lbmgpu_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw DeviceError(std::string("cannot load libnccl.so.2: ") + dlerror());
    using Fn = int (*)(void*);
    auto fn = reinterpret_cast<Fn>(dlsym(h, "ncclGetUniqueId"));
    if (!fn) throw DeviceError("libnccl.so.2 has no ncclGetUniqueId");
    if (fn(out128) != 0) throw DeviceError("ncclGetUniqueId failed");
  });
}

int lbmgpu_peer_export(lbmgpu_ctx* c, void* out, size_t cap, size_t* len) {
  return guard([&] {
    need(c, "ctx");
    need(len, "len");
    std::vector<uint8_t> rec;
    c->eng->peer_export(rec);
    *len = rec.size();
    if (out) {
      if (cap < rec.size()) throw ConfigError("peer transport: record buffer too small");
      std::memcpy(out, rec.data(), rec.size());
    }
  });
}

int lbmgpu_peer_attach(lbmgpu_ctx* c, const void* recs, size_t rec_len, int nranks) {
  return guard([&] {
    need(c, "ctx");
    need(recs, "records");
    c->eng->peer_attach(static_cast<const uint8_t*>(recs), rec_len, nranks);
  });
}

int lbmgpu_peer_probe(lbmgpu_ctx* c, int which, double* out, uint64_t count) {
  return guard([&] {
    need(c, "ctx");
    need(out, "out");
    std::vector<double> v;
    c->eng->peer_probe(which, v);
    if (count != v.size())
      throw ConfigError("peer probe: buffer holds " + std::to_string(count) + " values, plane has " +
                        std::to_string(v.size()));
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int lbmgpu_part_info(lbmgpu_ctx* c, int part, int* z0, int* z1, uint64_t* nf) {
  return guard([&] {
    need(c, "ctx");
    if (part < 0 || part >= c->eng->parts()) throw ConfigError("part out of range");
    int a = 0, b = 0;
    uint64_t n = 0;
    c->eng->part_info(part, &a, &b, &n);
    if (z0) *z0 = a;
    if (z1) *z1 = b;
    if (nf) *nf = n;
  });
}

int lbmgpu_halo_plan(int nz, int parts, int ring, int64_t* rows, int cap,
                     int* n_rows) {
  return guard([&] {
    if (nz < 1 || parts < 1 || parts > nz) throw ConfigError("halo_plan: bad nz/parts");
    if (ring < 0 || ring > 2) throw ConfigError("halo_plan: z_wrap must be 0, 1 or 2");
    std::vector<HaloRow> plan = ring == 2 ? halo_plan_os(nz, parts) : halo_plan(nz, parts, ring != 0);
    if (n_rows) *n_rows = static_cast<int>(plan.size());
    for (int i = 0; i < cap && i < static_cast<int>(plan.size()); ++i) {
      const HaloRow& r = plan[i];
      int64_t* o = rows + 7 * i;
      o[0] = r.phase;
      o[1] = r.src_part;
      o[2] = r.dst_part;
      o[3] = r.src_plane;
      o[4] = r.dst_plane;
      o[5] = r.slot0;
      o[6] = kHaloSlots;
    }
  });
}

}  // extern "C"

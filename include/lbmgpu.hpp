// lbmgpu.hpp -- header-only C++ host API over the C ABI (include/lbmgpu.h).
//
// Mirrors the reference lbmbench surface (paths relative to
// /root/reference/proj) so a caller of the reference can switch by changing
// the namespace:
//   lbm::TrtParams / BodyForce          include/lbm/d3q19.hpp:64-92
//   lbm::GeometrySpec                   include/lbm/geometry.hpp:36-42
//   lbm::PaddingPolicy                  include/lbm/list_lattice.hpp:25-39
//   lbm::KernelDescriptor               include/lbm/kernels.hpp:25-36
//   lbm::Kernel / make_kernel           include/lbm/kernels.hpp:58-105
//   lbm::ConfigError / NumericalError   include/lbm/errors.hpp:9-18
//   state_fingerprint / perturbed_equilibrium  src/harness.cpp:27-62
//   verify_kernel                       src/verification.cpp:31-100
// Every compute call runs on the GPU through liblbmgpu.so.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbmgpu.h"

namespace lbmgpu {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc) {
  if (rc == LBMGPU_OK) return;
  const std::string msg = lbmgpu_last_error();
  if (rc == LBMGPU_ECONFIG) throw ConfigError(msg);
  if (rc == LBMGPU_ENUMERICAL) throw NumericalError(msg);
  throw DeviceError(msg);
}

inline constexpr int kQ = 19;

struct TrtParams {
  double omega_plus = 1.0;
  double magic_lambda = 3.0 / 16.0;
  double viscosity() const { return (1.0 / omega_plus - 0.5) / 3.0; }
  double omega_minus() const { return lbmgpu_omega_minus(omega_plus, magic_lambda); }
  static TrtParams from_tau(double tau_plus, double lambda = 3.0 / 16.0) {
    return TrtParams{1.0 / tau_plus, lambda};
  }
};

struct BodyForce {
  std::array<double, 3> g = {0.0, 0.0, 0.0};
};

enum class GeometryKind { Channel = 0, Slit = 1, Pipe = 2, Blocks = 3 };

inline const char* to_string(GeometryKind k) {
  switch (k) {
    case GeometryKind::Channel: return "channel";
    case GeometryKind::Slit: return "slit";
    case GeometryKind::Pipe: return "pipe";
    case GeometryKind::Blocks: return "blocks";
  }
  return "?";
}

inline GeometryKind geometry_kind_from_string(const std::string& s) {
  if (s == "channel") return GeometryKind::Channel;
  if (s == "slit") return GeometryKind::Slit;
  if (s == "pipe") return GeometryKind::Pipe;
  if (s == "blocks") return GeometryKind::Blocks;
  throw ConfigError("unknown geometry kind '" + s + "' (valid: channel, slit, pipe, blocks)");
}

struct GeometrySpec {
  GeometryKind kind = GeometryKind::Channel;
  int nx = 500, ny = 100, nz = 100;
  int block = 4, spacing = 4;
  int pipe_diameter = 0;  // extension: 0 = reference D = min(ny,nz)-2

  lbmgpu_geometry c() const {
    lbmgpu_geometry g{};
    g.kind = static_cast<int>(kind);
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.block = block;
    g.spacing = spacing;
    g.pipe_diameter = pipe_diameter;
    return g;
  }
};

struct PaddingPolicy {
  enum class Mode { None = 0, Auto = 1, Thrash = 2, Explicit = 3 };
  Mode mode = Mode::None;
  std::array<std::int64_t, kQ> pads{};
  static PaddingPolicy none() { return {}; }
  static PaddingPolicy automatic() { return {Mode::Auto, {}}; }
  static PaddingPolicy thrash() { return {Mode::Thrash, {}}; }

  // list_lattice.cpp:10-34
  static PaddingPolicy parse(const std::string& s) {
    if (s == "none") return none();
    if (s == "auto") return automatic();
    if (s == "thrash") return thrash();
    PaddingPolicy p{Mode::Explicit, {}};
    size_t pos = 0;
    int n = 0;
    while (pos <= s.size() && n < kQ) {
      const size_t e = s.find(',', pos);
      const std::string item = s.substr(pos, e == std::string::npos ? std::string::npos : e - pos);
      try {
        p.pads[n] = std::stoll(item);
      } catch (...) {
        throw ConfigError("padding: cannot parse pad count '" + item +
                          "' (example: --padding auto)");
      }
      if (p.pads[n] < 0) throw ConfigError("padding: pad counts must be >= 0");
      ++n;
      if (e == std::string::npos) break;
      pos = e + 1;
    }
    if (n != kQ)
      throw ConfigError("padding: expected 'none', 'auto', 'thrash' or 19 comma-separated pad "
                        "counts (example: --padding auto)");
    return p;
  }
  std::string to_string() const {
    switch (mode) {
      case Mode::None: return "none";
      case Mode::Auto: return "auto";
      case Mode::Thrash: return "thrash";
      case Mode::Explicit: {
        std::string o;
        for (int i = 0; i < kQ; ++i) o += (i ? "," : "") + std::to_string(pads[i]);
        return o;
      }
    }
    return "?";
  }
  lbmgpu_padding c() const {
    lbmgpu_padding p{};
    p.mode = static_cast<int>(mode);
    for (int d = 0; d < kQ; ++d) p.pads[d] = pads[d];
    return p;
  }
};

enum class Propagation { OsPush = 0, OsPull = 1, Aa = 2 };
enum class Addressing { Direct, Indirect };
enum class Layout { AoS, SoA };

struct KernelDescriptor {
  std::string name;
  Propagation prop = Propagation::OsPush;
  Layout layout = Layout::SoA;
  Addressing addr = Addressing::Direct;
  int blk = 0;
  int nt_streams = 0;
  bool ria = false, pv = false, vec = false;
  int vector_width = 4;
};

inline std::vector<std::string> kernel_names() {
  char buf[2048];
  check(lbmgpu_kernel_names(buf, sizeof(buf)));
  std::vector<std::string> out;
  std::string cur;
  for (const char* p = buf; *p; ++p) {
    if (*p == '\n') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += *p;
    }
  }
  return out;
}

inline KernelDescriptor make_descriptor(const std::string& name, int blk = 0,
                                        int vector_width = 4) {
  lbmgpu_descriptor c{};
  check(lbmgpu_make_descriptor(name.c_str(), blk, vector_width, &c));
  KernelDescriptor d;
  d.name = name;
  d.prop = static_cast<Propagation>(c.prop);
  d.layout = c.layout_soa ? Layout::SoA : Layout::AoS;
  d.addr = c.indirect ? Addressing::Indirect : Addressing::Direct;
  d.blk = c.blk;
  d.nt_streams = c.nt_streams;
  d.ria = c.ria;
  d.pv = c.pv;
  d.vec = c.vec;
  d.vector_width = c.vector_width;
  return d;
}

struct KernelCaps {
  bool nt_stores_available = false;
  int nt_streams_effective = 0;
  bool huge_pages_advised = false;
};

struct RiaStats {
  std::size_t total_runs = 0;
  std::size_t n_fluid = 0;
};

// GPU-resident kernel + lattice; the reference lbm::Kernel contract.
class Kernel {
 public:
  Kernel(const KernelDescriptor& d, const GeometrySpec& g, const PaddingPolicy& pad,
         int row_pad = 0, const lbmgpu_dist* dist = nullptr)
      : desc_(d) {
    const lbmgpu_geometry gc = g.c();
    const lbmgpu_padding pc = pad.c();
    lbmgpu_ctx* raw = nullptr;
    check(lbmgpu_create(d.name.c_str(), d.blk, d.vector_width, &gc, &pc, row_pad, dist, &raw));
    ctx_.reset(raw);
  }

  const KernelDescriptor& descriptor() const { return desc_; }
  lbmgpu_ctx* handle() const { return ctx_.get(); }

  void advance(const TrtParams& p, const BodyForce& g, long steps) {
    check(lbmgpu_advance(ctx_.get(), p.omega_plus, p.magic_lambda, g.g.data(), steps));
  }
  // advance() bracketed by CUDA events on the kernel's stream; device ms.
  double time_advance(const TrtParams& p, const BodyForce& g, long steps) {
    double ms = 0;
    check(lbmgpu_time_advance(ctx_.get(), p.omega_plus, p.magic_lambda, g.g.data(), steps, &ms));
    return ms;
  }
  std::size_t n_fluid() const {
    std::uint64_t n = 0;
    check(lbmgpu_n_fluid(ctx_.get(), &n));
    return n;
  }
  KernelCaps capabilities() const {
    int a = 0, b = 0, c = 0;
    check(lbmgpu_capabilities(ctx_.get(), &a, &b, &c));
    return {a != 0, b, c != 0};
  }
  std::vector<double> snapshot() const {
    std::vector<double> out(n_fluid() * kQ);
    check(lbmgpu_snapshot(ctx_.get(), out.data(), out.size()));
    return out;
  }
  void load_state(std::span<const double> s) {
    check(lbmgpu_load_state(ctx_.get(), s.data(), s.size()));
  }
  // load_state(in) + advance(steps) + snapshot(out) as one job (lbmgpu_run);
  // returns whether the transfers were pipelined with the sweeps.
  bool run(std::span<const double> in, const TrtParams& p, const BodyForce& g, long steps,
           std::span<double> out) {
    int piped = 0;
    check(lbmgpu_run(ctx_.get(), p.omega_plus, p.magic_lambda, g.g.data(), steps, in.data(),
                     in.size(), out.data(), out.size(), &piped));
    return piped != 0;
  }
  void load_perturbed(std::uint64_t seed, double amplitude = 1e-3) {
    check(lbmgpu_load_perturbed(ctx_.get(), seed, amplitude));
  }
  double total_mass() const {
    double m = 0;
    check(lbmgpu_total_mass(ctx_.get(), &m));
    return m;
  }
  std::uint64_t fingerprint() const {
    std::uint64_t h = 0;
    check(lbmgpu_fingerprint(ctx_.get(), &h));
    return h;
  }
  std::optional<RiaStats> ria_stats() const {
    std::int64_t r = 0, n = 0;
    double v = 0, pv = 0;
    check(lbmgpu_ria_stats(ctx_.get(), &r, &n, &v, &pv));
    if (r < 0) return std::nullopt;
    return RiaStats{static_cast<std::size_t>(r), static_cast<std::size_t>(n)};
  }
  std::optional<double> vector_fraction() const {
    std::int64_t r = 0, n = 0;
    double v = 0, pv = 0;
    check(lbmgpu_ria_stats(ctx_.get(), &r, &n, &v, &pv));
    if (v < 0) return std::nullopt;
    return v;
  }
  std::optional<double> pv_chunk_fraction() const {
    std::int64_t r = 0, n = 0;
    double v = 0, pv = 0;
    check(lbmgpu_ria_stats(ctx_.get(), &r, &n, &v, &pv));
    if (pv < 0) return std::nullopt;
    return pv;
  }
  // vectorizable_fraction(coding, W) (list_lattice.cpp:228-236) at any width
  std::optional<double> vectorizable_fraction(int width) const {
    double v = 0;
    check(lbmgpu_vectorizable_fraction(ctx_.get(), width, &v));
    if (v < 0) return std::nullopt;
    return v;
  }
  // run starts of the run coding (RiaRun::start), node order; empty without a coding
  std::vector<std::uint32_t> export_runs() const {
    std::int64_t n = 0;
    check(lbmgpu_export_runs(ctx_.get(), nullptr, 0, &n));
    std::vector<std::uint32_t> r(n > 0 ? static_cast<std::size_t>(n) : 0);
    if (n > 0) check(lbmgpu_export_runs(ctx_.get(), r.data(), r.size(), &n));
    return r;
  }
  // Peer-memory transport (lbmgpu_dist.transport = 1, nranks > 1): this
  // rank's CUDA IPC record; all-gather them and pass all ranks' records
  // (rank order) to peer_attach before the first advance.
  std::vector<std::uint8_t> peer_export() const {
    std::size_t len = 0;
    check(lbmgpu_peer_export(ctx_.get(), nullptr, 0, &len));
    std::vector<std::uint8_t> rec(len);
    check(lbmgpu_peer_export(ctx_.get(), rec.data(), rec.size(), &len));
    return rec;
  }
  void peer_attach(std::span<const std::uint8_t> records, int nranks) {
    check(lbmgpu_peer_attach(ctx_.get(), records.data(),
                             nranks > 0 ? records.size() / nranks : 0, nranks));
  }

 private:
  struct Del {
    void operator()(lbmgpu_ctx* c) const { lbmgpu_destroy(c); }
  };
  KernelDescriptor desc_;
  std::unique_ptr<lbmgpu_ctx, Del> ctx_;
};

inline std::unique_ptr<Kernel> make_kernel(const KernelDescriptor& d, const GeometrySpec& g,
                                           const PaddingPolicy& pad = PaddingPolicy::automatic(),
                                           int row_pad = 0) {
  return std::make_unique<Kernel>(d, g, pad, row_pad);
}

inline std::uint64_t state_fingerprint(const std::vector<double>& snapshot) {
  return lbmgpu_fnv1a(snapshot.data(), snapshot.size() * sizeof(double));
}

struct LoopBalance {
  double ref_min = 0, ref_max = 0, gpu = 0;
};
inline LoopBalance loop_balance(const std::string& name) {
  LoopBalance b;
  check(lbmgpu_loop_balance(name.c_str(), &b.ref_min, &b.ref_max, &b.gpu));
  return b;
}

// loop_balance(desc, RiaStats) (perfmodel.cpp:21-31)
inline LoopBalance loop_balance(const std::string& name, std::int64_t total_runs,
                                std::int64_t n_fluid) {
  LoopBalance b;
  check(lbmgpu_loop_balance_stats(name.c_str(), total_runs, n_fluid, &b.ref_min, &b.ref_max,
                                  &b.gpu));
  return b;
}
// roofline (perfmodel.cpp:73-87)
struct RooflinePrediction {
  double gbps = 0, min_bflup = 0, max_bflup = 0, pmax_min_mflups = 0, pmax_max_mflups = 0;
};
inline RooflinePrediction roofline(double gbps, double bl_min, double bl_max) {
  RooflinePrediction r;
  r.gbps = gbps;
  r.min_bflup = bl_min;
  r.max_bflup = bl_max;
  check(lbmgpu_roofline(gbps, bl_min, bl_max, &r.pmax_min_mflups, &r.pmax_max_mflups));
  return r;
}

// Device bandwidth micro-benchmarks (run_microbench, microbench.cpp:57-175)
// and which of them models which kernel (micro_for, perfmodel.cpp:66-71).
inline double microbench(const std::string& kind, std::uint64_t working_set_bytes, int reps = 5) {
  double gbps = 0;
  check(lbmgpu_microbench(kind.c_str(), working_set_bytes, reps, &gbps));
  return gbps;
}
inline const char* micro_for(const KernelDescriptor& k) {
  if (k.nt_streams > 0) return "copy-19-nt-sl";
  if (k.prop == Propagation::Aa) return "update-19";
  return "copy-19";
}

struct PoiseuilleCase {
  int nx = 8, ny = 8, nz = 34;
  double g = 1e-6;
  TrtParams params = TrtParams::from_tau(0.9);
};

struct VerificationReport {
  std::string kernel;
  PoiseuilleCase setup;
  std::vector<double> simulated, analytic;
  double half_force_shift = 0, linf_rel = 0, l2_rel = 0;
  long steps = 0;
  bool converged = false, passed = false;
};

inline constexpr double kVerifyLinfTolerance = 1e-4;

inline VerificationReport verify_kernel(const KernelDescriptor& k, const PoiseuilleCase& c,
                                        long check_interval = 200, double rel_tol = 1e-12,
                                        long max_steps = 200000) {
  VerificationReport r;
  r.kernel = k.name;
  r.setup = c;
  const int layers = c.nz - 2;
  r.simulated.assign(layers > 0 ? layers : 0, 0.0);
  r.analytic.assign(layers > 0 ? layers : 0, 0.0);
  lbmgpu_verify_report rep{};
  check(lbmgpu_verify(k.name.c_str(), c.nx, c.ny, c.nz, c.g, 1.0 / c.params.omega_plus,
                      c.params.magic_lambda, check_interval, rel_tol, max_steps, &rep,
                      r.simulated.data(), r.analytic.data()));
  r.half_force_shift = rep.half_force_shift;
  r.linf_rel = rep.linf_rel;
  r.l2_rel = rep.l2_rel;
  r.steps = rep.steps;
  r.converged = rep.converged != 0;
  r.passed = rep.passed != 0;
  return r;
}

}  // namespace lbmgpu

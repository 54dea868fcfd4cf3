// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C-ABI driver around the UNMODIFIED reference library (lbmbench, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// exposes exactly the oracle path SURVEY.md section 3E names:
//   build_geometry -> WorkerPool(N) -> make_kernel(make_descriptor(name), ff,
//   padding, pool) -> load_state / advance / snapshot / total_mass
// plus build_structure / padding_offsets / perturbed_equilibrium /
// state_fingerprint / verify_kernel / loop_balance for the bit-exact checks.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
// --impl reference legs load this library, and only as the checker / the
// reference CPU arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lbm/errors.hpp"
#include "lbm/geometry.hpp"
#include "lbm/harness.hpp"
#include "lbm/kernels.hpp"
#include "lbm/microbench.hpp"
#include "lbm/list_lattice.hpp"
#include "lbm/perfmodel.hpp"
#include "lbm/verification.hpp"
#include "lbm/workers.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const lbm::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const lbm::NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// kind: 0 channel, 1 slit, 2 pipe, 3 blocks (the order of lbm::GeometryKind).
// pipe_diameter > 0 hand-builds the pipe with the reference's own staircase
// test 4((y-cy)^2+(z-cz)^2) > D^2 (geometry.cpp:68-84 with D = min(ny,nz)-2
// being the stock case); make_kernel accepts any FlagField.
lbm::FlagField make_flags(int kind, int nx, int ny, int nz, int block,
                          int spacing, int pipe_diameter) {
  lbm::GeometrySpec s;
  s.kind = static_cast<lbm::GeometryKind>(kind);
  s.nx = nx;
  s.ny = ny;
  s.nz = nz;
  s.block = block;
  s.spacing = spacing;
  lbm::FlagField ff = lbm::build_geometry(s);
  if (s.kind == lbm::GeometryKind::Pipe && pipe_diameter > 0) {
    const std::int64_t d2 =
        static_cast<std::int64_t>(pipe_diameter) * pipe_diameter;
    for (int y = 0; y < ny; ++y)
      for (int z = 0; z < nz; ++z) {
        const std::int64_t dy = 2 * y - (ny - 1);
        const std::int64_t dz = 2 * z - (nz - 1);
        const std::uint8_t v = (dy * dy + dz * dz > d2) ? 1 : 0;
        for (int x = 0; x < nx; ++x) ff.flags[ff.index(x, y, z)] = v;
      }
    if (lbm::fluid_count(ff) == 0)
      throw lbm::ConfigError("pipe: diameter leaves no fluid");
  }
  return ff;
}

lbm::PaddingPolicy make_padding(int mode, const std::int64_t* pads) {
  lbm::PaddingPolicy p;
  switch (mode) {
    case 0: p = lbm::PaddingPolicy::none(); break;
    case 1: p = lbm::PaddingPolicy::automatic(); break;
    case 2: p = lbm::PaddingPolicy::thrash(); break;
    case 3:
      p.mode = lbm::PaddingPolicy::Mode::Explicit;
      for (int d = 0; d < lbm::kQ; ++d) p.pads[d] = pads[d];
      break;
    default: throw lbm::ConfigError("bad padding mode");
  }
  return p;
}

struct Handle {
  lbm::FlagField ff;
  std::unique_ptr<lbm::WorkerPool> pool;
  std::unique_ptr<lbm::Kernel> kernel;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_geometry(int kind, int nx, int ny, int nz, int block, int spacing,
                 int pipe_diameter, std::uint8_t* flags_out,
                 std::int64_t* n_fluid, int* periodic_out) {
  return guard([&] {
    lbm::FlagField ff =
        make_flags(kind, nx, ny, nz, block, spacing, pipe_diameter);
    if (flags_out) std::memcpy(flags_out, ff.flags.data(), ff.flags.size());
    if (n_fluid) *n_fluid = lbm::fluid_count(ff);
    if (periodic_out)
      for (int a = 0; a < 3; ++a) periodic_out[a] = ff.periodic[a];
  });
}

// pin / npin: core ids for the workers (reference --pin semantics,
// workers.cpp:26-39: worker w is bound to pin[w]); npin = 0 leaves them
// unpinned.
int ref_create(const char* name, int kind, int nx, int ny, int nz, int block,
               int spacing, int pipe_diameter, int blk, int pad_mode,
               const std::int64_t* pads, int threads, int vector_width,
               const int* pin, int npin, void** out) {
  return guard([&] {
    auto h = std::make_unique<Handle>();
    h->ff = make_flags(kind, nx, ny, nz, block, spacing, pipe_diameter);
    h->pool = std::make_unique<lbm::WorkerPool>(
        threads, npin > 0 ? std::vector<int>(pin, pin + npin) : std::vector<int>{});
    h->kernel = lbm::make_kernel(lbm::make_descriptor(name, blk, vector_width),
                                 h->ff, make_padding(pad_mode, pads),
                                 *h->pool);
    *out = h.release();
  });
}

void ref_destroy(void* h) { delete static_cast<Handle*>(h); }

// One repetition of the reference's run_microbench (microbench.cpp:57-175)
// with the shortest protocol: bytes accounted per pass and passes, for the
// accounting check against lbmgpu_microbench_accounting.
int ref_microbench(const char* kind, std::uint64_t working_set, int workers,
                   std::uint64_t* bytes_per_pass, int* passes, double* gbps) {
  return guard([&] {
    lbm::MicrobenchProtocol proto;
    proto.min_seconds = 0.0;
    proto.repetitions = 1;
    const lbm::BandwidthMeasurement m =
        lbm::run_microbench(lbm::micro_kind_from_string(kind), working_set, workers, proto);
    *bytes_per_pass = m.passes ? m.bytes_accounted / m.passes : 0;
    *passes = m.passes;
    *gbps = m.gbps;
  });
}

std::uint64_t ref_llc_bytes(void) { return lbm::detect_llc_bytes(); }

// number of workers whose core binding was applied
int ref_pinned(void* h, int* out) {
  return guard([&] {
    int n = 0;
    for (const auto& a : static_cast<Handle*>(h)->pool->affinity()) n += a.applied ? 1 : 0;
    *out = n;
  });
}

int ref_n_fluid(void* h, std::uint64_t* out) {
  return guard([&] { *out = static_cast<Handle*>(h)->kernel->n_fluid(); });
}

int ref_load_state(void* h, const double* state, std::uint64_t count) {
  return guard([&] {
    static_cast<Handle*>(h)->kernel->load_state(
        std::span<const double>(state, count));
  });
}

int ref_snapshot(void* h, double* out, std::uint64_t count) {
  return guard([&] {
    const std::vector<double> s = static_cast<Handle*>(h)->kernel->snapshot();
    if (s.size() != count) throw lbm::ConfigError("snapshot size mismatch");
    std::memcpy(out, s.data(), count * sizeof(double));
  });
}

int ref_fingerprint_state(void* h, std::uint64_t* out) {
  return guard([&] {
    *out = lbm::state_fingerprint(static_cast<Handle*>(h)->kernel->snapshot());
  });
}

int ref_total_mass(void* h, double* out) {
  return guard([&] { *out = static_cast<Handle*>(h)->kernel->total_mass(); });
}

// omega_plus / magic_lambda exactly as TrtParams (d3q19.hpp:64-86).
int ref_advance(void* h, double omega_plus, double magic_lambda,
                const double* g, long steps, double* seconds) {
  return guard([&] {
    lbm::TrtParams p{omega_plus, magic_lambda};
    lbm::BodyForce f{{g[0], g[1], g[2]}};
    const auto t0 = std::chrono::steady_clock::now();
    static_cast<Handle*>(h)->kernel->advance(p, f, steps);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

int ref_ria_stats(void* h, std::uint64_t* runs, double* vfrac) {
  return guard([&] {
    auto* k = static_cast<Handle*>(h)->kernel.get();
    auto st = k->ria_stats();
    *runs = st ? st->total_runs : 0;
    auto v = k->vector_fraction();
    *vfrac = v ? *v : -1.0;
  });
}

// Structure export: nodes (3 int32 per node), adjacency [n*18+d-1] (u32),
// starts[19] and total slots.  Pass nulls to query n_fluid only.
int ref_structure(int kind, int nx, int ny, int nz, int block, int spacing,
                  int pipe_diameter, int layout_soa, int blk, int pad_mode,
                  const std::int64_t* pads, int scatter, std::uint64_t* n_fluid,
                  std::int32_t* nodes_out, std::uint32_t* adj_out,
                  std::uint64_t* starts_out, std::uint64_t* total_slots) {
  return guard([&] {
    lbm::FlagField ff =
        make_flags(kind, nx, ny, nz, block, spacing, pipe_diameter);
    lbm::ListStructure ls = lbm::build_structure(
        ff, layout_soa ? lbm::Layout::SoA : lbm::Layout::AoS, blk,
        make_padding(pad_mode, pads),
        scatter ? lbm::Orientation::Scatter : lbm::Orientation::Gather);
    *n_fluid = ls.n_fluid;
    if (nodes_out)
      for (std::size_t n = 0; n < ls.n_fluid; ++n) {
        nodes_out[3 * n] = ls.nodes[n].x;
        nodes_out[3 * n + 1] = ls.nodes[n].y;
        nodes_out[3 * n + 2] = ls.nodes[n].z;
      }
    if (adj_out)
      std::memcpy(adj_out, ls.adj.data(), ls.n_fluid * 18 * sizeof(std::uint32_t));
    if (starts_out)
      for (int d = 0; d < lbm::kQ; ++d) starts_out[d] = ls.slots.starts[d];
    if (total_slots) *total_slots = ls.slots.total_slots;
  });
}

int ref_ria(int kind, int nx, int ny, int nz, int block, int spacing, int blk,
            int vector_width, std::uint64_t* runs, double* vfrac) {
  return guard([&] {
    lbm::FlagField ff = make_flags(kind, nx, ny, nz, block, spacing, 0);
    lbm::ListStructure ls =
        lbm::build_structure(ff, lbm::Layout::SoA, blk,
                             lbm::PaddingPolicy::none(),
                             lbm::Orientation::Scatter);
    lbm::RiaCoding r = lbm::build_ria(ls);
    *runs = r.total_runs();
    *vfrac = lbm::vectorizable_fraction(r, vector_width);
  });
}

int ref_padding_offsets(std::uint64_t n_fluid, int pad_mode,
                        const std::int64_t* pads, std::uint64_t* starts,
                        std::uint64_t* total) {
  return guard([&] {
    std::size_t tot = 0;
    auto s = lbm::padding_offsets(n_fluid, make_padding(pad_mode, pads), &tot);
    for (int d = 0; d < lbm::kQ; ++d) starts[d] = s[d];
    *total = tot;
  });
}

int ref_perturbed(std::uint64_t n_fluid, std::uint64_t seed, double amplitude,
                  double* out) {
  return guard([&] {
    auto v = lbm::perturbed_equilibrium(n_fluid, seed, amplitude);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

std::uint64_t ref_fingerprint(const double* data, std::uint64_t count) {
  return lbm::state_fingerprint(std::vector<double>(data, data + count));
}

void ref_collide_node(double* f, double wp, double wm, const double* g) {
  lbm::collide_node(f, wp, wm, g);
}

int ref_descriptor(const char* name, int blk, int* prop, int* layout_soa,
                   int* indirect, int* nt, int* ria, int* pv, int* vec) {
  return guard([&] {
    lbm::KernelDescriptor d = lbm::make_descriptor(name, blk);
    *prop = static_cast<int>(d.prop);
    *layout_soa = d.layout == lbm::Layout::SoA;
    *indirect = d.addr == lbm::Addressing::Indirect;
    *nt = d.nt_streams;
    *ria = d.ria;
    *pv = d.pv;
    *vec = d.vec;
  });
}

int ref_loop_balance(const char* name, double* bl_min, double* bl_max) {
  return guard([&] {
    lbm::LoopBalance b = lbm::loop_balance(lbm::make_descriptor(name));
    *bl_min = b.min_bflup;
    *bl_max = b.max_bflup;
  });
}

int ref_kernel_names(char* buf, std::uint64_t cap) {
  return guard([&] {
    std::string s;
    for (const auto& n : lbm::kernel_names()) s += n + "\n";
    if (s.size() + 1 > cap) throw lbm::ConfigError("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int ref_verify(const char* name, int nx, int ny, int nz, double g, double tau,
               double magic_lambda, int threads, long interval, double tol,
               long max_steps, double* linf, double* l2, long* steps,
               int* converged, int* passed, double* simulated,
               double* analytic) {
  return guard([&] {
    lbm::PoiseuilleCase c;
    c.nx = nx;
    c.ny = ny;
    c.nz = nz;
    c.g = g;
    c.params = lbm::TrtParams::from_tau(tau, magic_lambda);
    lbm::VerificationReport r = lbm::verify_kernel(
        lbm::make_descriptor(name), c, threads, interval, tol, max_steps);
    *linf = r.linf_rel;
    *l2 = r.l2_rel;
    *steps = r.steps;
    *converged = r.converged;
    *passed = r.passed;
    if (simulated)
      std::memcpy(simulated, r.simulated.data(),
                  r.simulated.size() * sizeof(double));
    if (analytic)
      std::memcpy(analytic, r.analytic.data(),
                  r.analytic.size() * sizeof(double));
  });
}

}  // extern "C"

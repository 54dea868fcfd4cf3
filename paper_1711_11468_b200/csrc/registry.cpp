// Kernel registry, descriptor parsing, padding and loop balance.
// Host-only restatements of the reference's registry layer (L5) -- these are
// the names and error messages a drop-in must keep.
#include <algorithm>

#include "lbm.hpp"

#include <cstdlib>
#include <map>
#include <mutex>

namespace lbmgpu {

// kernel_names() (reference src/kernels.cpp:22-43), canonical order.
const std::vector<std::string>& kernel_names() {
  static const std::vector<std::string> names = {
      "blk-push-aos",   "blk-push-soa",   "blk-pull-aos",
      "blk-pull-soa",   "aa-aos",         "aa-soa",
      "aa-vec-soa",     "list-push-aos",  "list-push-soa",
      "list-pull-aos",  "list-pull-soa",  "list-pull-split-nt-1s-soa",
      "list-pull-split-nt-2s-soa",        "list-aa-aos",
      "list-aa-soa",    "list-aa-ria-soa", "list-aa-pv-soa",
  };
  return names;
}

static bool ends_with(const std::string& s, const std::string& t) {
  return s.size() >= t.size() && s.compare(s.size() - t.size(), t.size(), t) == 0;
}
static bool starts_with(const std::string& s, const std::string& t) {
  return s.compare(0, t.size(), t) == 0;
}

// make_descriptor (reference src/kernels.cpp:50-82)
Descriptor make_descriptor(const std::string& name, int blk, int W) {
  const auto& names = kernel_names();
  if (std::find(names.begin(), names.end(), name) == names.end()) {
    std::string msg = "unknown kernel '" + name + "'; valid kernels:";
    for (const auto& n : names) msg += "\n  " + n;
    throw ConfigError(msg);
  }
  if (blk < 0) throw ConfigError("--blk must be >= 0, e.g. --blk 8");
  if (W < 1 || W > 8) throw ConfigError("vector width must be in [1, 8]");
  Descriptor d;
  d.name = name;
  d.blk = blk;
  d.vector_width = W;
  d.soa = !ends_with(name, "aos");
  d.indirect = starts_with(name, "list-");
  if (name.find("push") != std::string::npos)
    d.prop = Prop::OsPush;
  else if (name.find("pull") != std::string::npos)
    d.prop = Prop::OsPull;
  else
    d.prop = Prop::Aa;
  if (name.find("nt-1s") != std::string::npos) d.nt_streams = 1;
  if (name.find("nt-2s") != std::string::npos) d.nt_streams = 2;
  d.vec = name == "aa-vec-soa";
  d.ria = name == "list-aa-ria-soa" || name == "list-aa-pv-soa";
  d.pv = name == "list-aa-pv-soa";
  return d;
}

// loop_balance (reference src/perfmodel.cpp:10-47), plus the GPU algorithmic
// bytes: 19 PDF reads + 19 writes of 8 B (no write allocate on the GPU),
// + 18 x 4 B adjacency per one-step list update, or per odd AA sub-step
// (half of it per update), 0.5 B for the RIA names' pattern ids.  Reference
// side of the RIA names: without geometry statistics the index range is
// [0, 38] B; with them (total_runs >= 0, n_fluid > 0) both ends are the 76 B
// of run metadata amortised over the run and the even/odd pair, clamped to
// [0, 38] (perfmodel.cpp:21-31).
LoopBalance loop_balance(const Descriptor& k, int64_t total_runs, int64_t n_fluid) {
  LoopBalance b;
  const double rd = 8.0 * kQ, wr = 8.0 * kQ;
  const bool os = k.prop != Prop::Aa;
  const bool nt = k.nt_streams > 0;
  const double wa = (os && !nt) ? 8.0 * kQ : 0.0;
  double imin = 0, imax = 0, igpu = 0;
  if (k.indirect) {
    if (k.ria) {
      if (total_runs >= 0 && n_fluid > 0) {
        const double per_flup =
            76.0 * static_cast<double>(total_runs) / (2.0 * static_cast<double>(n_fluid));
        imin = imax = std::min(std::max(per_flup, 0.0), 38.0);
      } else {
        imin = 0.0;
        imax = 38.0;
      }
    } else if (os) {
      imin = imax = 18.0 * 4.0;
    } else {
      imin = imax = 18.0 * 4.0 / 2.0;
    }
    igpu = os ? 18.0 * 4.0 : 18.0 * 4.0 / 2.0;
    // ria / pv: the odd sub-step reads a one-byte pattern id per node instead
    // of 72 B of adjacency (list_ria.cuh; 2- and 4-byte ids or the run table
    // where a geometry has more than 256 distinct rows: 305-306 B)
    if (k.ria) igpu = 1.0 / 2.0;
  }
  b.ref_min = rd + wr + wa + imin;
  b.ref_max = rd + wr + wa + imax;
  b.gpu = rd + wr + igpu;
  return b;
}

// roofline (reference src/perfmodel.cpp:73-87): P_max = bandwidth / B_l; the
// lower prediction comes from the larger balance.
Roofline roofline(double gbps, double bl_min, double bl_max) {
  if (!(gbps > 0.0))
    throw ConfigError("roofline: bandwidth must be positive, got " + std::to_string(gbps));
  if (!(bl_min > 0.0) || !(bl_max > 0.0))
    throw ConfigError("roofline: loop balance must be positive");
  Roofline r;
  r.pmax_min_mflups = gbps * 1000.0 / bl_max;
  r.pmax_max_mflups = gbps * 1000.0 / bl_min;
  return r;
}

// ---- padding (reference src/list_lattice.cpp:63-121) ----------------------
namespace {
constexpr uint64_t kSetPeriod = 64 * 512 / 8;  // 4096 elements
constexpr uint64_t kPageElems = (2u << 20) / 8;  // 262144 elements

uint64_t place(uint64_t floor, uint64_t want_set, uint64_t want_tlb) {
  const uint64_t res = want_set * (64 / 8);
  uint64_t cand = (floor <= res) ? res
                                 : (floor - res + kSetPeriod - 1) / kSetPeriod *
                                           kSetPeriod +
                                       res;
  while (cand / kPageElems % 4 != want_tlb) cand += kSetPeriod;
  return cand;
}
}  // namespace

std::array<uint64_t, kQ> padding_offsets(uint64_t n, const Padding& p,
                                         uint64_t* total) {
  std::array<uint64_t, kQ> s{};
  switch (p.mode) {
    case 0:
      for (int d = 0; d < kQ; ++d) s[d] = uint64_t(d) * n;
      break;
    case 3: {
      uint64_t off = 0;
      for (int d = 0; d < kQ; ++d) {
        if (p.pads[d] < 0) throw ConfigError("padding: pad counts must be >= 0");
        off += uint64_t(p.pads[d]);
        s[d] = off;
        off += n;
      }
      break;
    }
    case 1: {
      uint64_t floor = 0;
      for (int d = 0; d < kQ; ++d) {
        s[d] = place(floor, uint64_t(d) * (512 / kQ) % 512, uint64_t(d) % 4);
        floor = s[d] + n;
      }
      break;
    }
    case 2: {
      uint64_t floor = 0;
      for (int d = 0; d < kQ; ++d) {
        s[d] = place(floor, 0, 0);
        floor = s[d] + n;
      }
      break;
    }
    default:
      throw ConfigError("padding: unknown mode");
  }
  if (total) *total = s[kQ - 1] + n;
  return s;
}

// ---- geometry argument checks (reference src/geometry.cpp:17-25,40-111) ----
static void check_dims(const GeomSpec& s, const char* kind, int mx, int my,
                       int mz) {
  if (s.nx < mx || s.ny < my || s.nz < mz)
    throw ConfigError(std::string("geometry '") + kind +
                      "' needs dims of at least " + std::to_string(mx) + "x" +
                      std::to_string(my) + "x" + std::to_string(mz) + ", got " +
                      std::to_string(s.nx) + "x" + std::to_string(s.ny) + "x" +
                      std::to_string(s.nz));
}

std::array<bool, 3> validate_geometry(const GeomSpec& s) {
  switch (s.kind) {
    case kChannel:
      check_dims(s, "channel", 1, 3, 3);
      return {true, false, false};
    case kSlit:
      check_dims(s, "slit", 1, 1, 3);
      return {true, true, false};
    case kPipe:
      check_dims(s, "pipe", 1, 4, 4);
      if (s.pipe_diameter < 0)
        throw ConfigError("pipe geometry: diameter must be >= 0");
      return {true, false, false};
    case kBlocks: {
      check_dims(s, "blocks", 1, 1, 1);
      if (s.block < 1)
        throw ConfigError("blocks geometry: block edge must be >= 1");
      if (s.spacing < 0)
        throw ConfigError("blocks geometry: spacing must be >= 0");
      const int period = s.block + s.spacing;
      if (period > std::min({s.nx, s.ny, s.nz}))
        throw ConfigError(
            "blocks geometry: block+spacing must not exceed the smallest "
            "dimension");
      return {true, true, true};
    }
    case kCustom:
      if (s.nx < 1 || s.ny < 1 || s.nz < 1)
        throw ConfigError("custom geometry: dims must be >= 1");
      if (s.custom.size() != s.volume())
        throw ConfigError("custom geometry: flag field size mismatch");
      return {s.custom_periodic[0], s.custom_periodic[1], s.custom_periodic[2]};
    default:
      throw ConfigError("unknown geometry kind (valid: channel, slit, pipe, blocks)");
  }
}

// ---- guard zones around device buffers (lbm.hpp) ---------------------------
namespace {
struct GuardRegistry {
  std::mutex m;
  std::map<void*, size_t> live;  // user pointer -> user bytes
  static GuardRegistry& get() {
    static GuardRegistry r;
    return r;
  }
};
}  // namespace

bool guard_enabled() {
  const char* e = std::getenv("LBMGPU_GUARD");
  return e && std::atoi(e) != 0;
}

void* guarded_malloc(size_t bytes) {
  const size_t user = (bytes + 255) / 256 * 256;  // keep the 256-byte alignment
  unsigned char* raw = nullptr;
  LBM_CUDA(cudaMalloc(reinterpret_cast<void**>(&raw), user + 2 * kGuardBytes));
  LBM_CUDA(cudaMemset(raw, kGuardByte, kGuardBytes));
  LBM_CUDA(cudaMemset(raw + kGuardBytes + user, kGuardByte, kGuardBytes));
  void* p = raw + kGuardBytes;
  GuardRegistry& r = GuardRegistry::get();
  std::lock_guard<std::mutex> lk(r.m);
  r.live[p] = user;
  return p;
}

void guarded_free(void* user) {
  GuardRegistry& r = GuardRegistry::get();
  {
    std::lock_guard<std::mutex> lk(r.m);
    r.live.erase(user);
  }
  cudaFree(static_cast<unsigned char*>(user) - kGuardBytes);
}

// Negative control of the guard zones: a guarded buffer written 8 bytes past
// its end must be reported (returns the count guard_check saw, then frees).
int guard_selftest() {
  unsigned char* p = static_cast<unsigned char*>(guarded_malloc(1000));
  LBM_CUDA(cudaMemset(p + 1024, 0, 8));  // user size rounds up to 1024
  const int bad = guard_check(nullptr);
  guarded_free(p);
  return bad;
}

int guard_check(std::string* report) {
  LBM_CUDA(cudaDeviceSynchronize());
  GuardRegistry& r = GuardRegistry::get();
  std::lock_guard<std::mutex> lk(r.m);
  std::vector<unsigned char> h(kGuardBytes);
  int bad = 0;
  for (const auto& [p, bytes] : r.live) {
    unsigned char* user = static_cast<unsigned char*>(p);
    for (int side = 0; side < 2; ++side) {
      const unsigned char* g = side ? user + bytes : user - kGuardBytes;
      LBM_CUDA(cudaMemcpy(h.data(), g, kGuardBytes, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < kGuardBytes; ++i)
        if (h[i] != kGuardByte) {
          ++bad;
          if (report)
            *report += std::string(side ? "after" : "before") + " buffer of " +
                       std::to_string(bytes) + " bytes at offset " + std::to_string(i) + "; ";
          break;
        }
    }
  }
  return bad;
}

}  // namespace lbmgpu

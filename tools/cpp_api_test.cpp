// C++ host-API checks over include/lbmgpu.hpp, written like the reference's
// doctest kernel tests (proj/tests/test_kernels.cpp) so an lbmbench user can
// read them side by side.  Built by tools/Makefile, run by
// tests/test_cpp_api.py (GPU) and prints "ALL PASSED".
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../include/lbmgpu.hpp"

using namespace lbmgpu;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static const TrtParams kParams = TrtParams::from_tau(0.9);
static const BodyForce kForce{{1e-5, 2e-6, -3e-6}};

static GeometrySpec bench_blocks() {
  GeometrySpec g;
  g.kind = GeometryKind::Blocks;
  g.nx = 12;
  g.ny = 10;
  g.nz = 10;
  g.block = 4;
  g.spacing = 4;
  return g;
}

// "registry lists exactly the 17 kernel names" (test_kernels.cpp:29-54)
static void registry() {
  CHECK(kernel_names().size() == 17);
  CHECK(throws<ConfigError>([] { make_descriptor("plain-push"); }));
  const KernelDescriptor nt = make_descriptor("list-pull-split-nt-2s-soa");
  CHECK(nt.prop == Propagation::OsPull && nt.addr == Addressing::Indirect && nt.nt_streams == 2);
  const KernelDescriptor pv = make_descriptor("list-aa-pv-soa");
  CHECK(pv.prop == Propagation::Aa && pv.ria && pv.pv);
}

// "uniform equilibrium is a fixed point of every kernel" (:56-67)
static void fixed_point() {
  const double w[19] = {1.0 / 3, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18, 1.0 / 18,
                        1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36,
                        1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36};
  for (const std::string& name : kernel_names()) {
    auto k = make_kernel(make_descriptor(name), bench_blocks());
    k->advance(kParams, BodyForce{}, 4);
    const std::vector<double> s = k->snapshot();
    bool ok = true;
    for (std::size_t n = 0; n < s.size() / 19; ++n)
      for (int d = 0; d < 19; ++d) ok = ok && std::abs(s[n * 19 + d] - w[d]) <= 1e-15;
    CHECK(ok);
  }
}

// "results are bitwise identical across ..." + golden fingerprint of the
// reference (tests/golden/small.json, blocks_12x10x10 full / half family)
static void golden(const char* full_fp, const char* half_fp) {
  for (const std::string& name : kernel_names()) {
    auto k = make_kernel(make_descriptor(name), bench_blocks());
    k->load_perturbed(1234);
    k->advance(kParams, kForce, 8);
    char buf[20];
    std::snprintf(buf, sizeof(buf), "%016llx",
                  static_cast<unsigned long long>(state_fingerprint(k->snapshot())));
    const bool list = name.rfind("list-", 0) == 0;
    if (std::string(buf) != (list ? half_fp : full_fp)) {
      std::printf("fingerprint %s: %s\n", name.c_str(), buf);
      ++failures;
    }
  }
}

// "AA kernels reject odd step counts before touching state" (:167-175)
static void rejections() {
  auto k = make_kernel(make_descriptor("list-aa-soa"), bench_blocks());
  const std::vector<double> before = k->snapshot();
  CHECK(throws<ConfigError>([&] { k->advance(kParams, kForce, 3); }));
  CHECK(k->snapshot() == before);
  CHECK(throws<ConfigError>([&] { k->advance(kParams, kForce, -2); }));
  GeometrySpec bad = bench_blocks();
  bad.block = 0;
  CHECK(throws<ConfigError>([&] { make_kernel(make_descriptor("aa-soa"), bad); }));
  // the peer transport needs nranks > 1 and a direct SoA z-slab split
  CHECK(throws<ConfigError>([&] { k->peer_export(); }));
  GeometrySpec small;
  small.nx = 16;
  small.ny = 12;
  small.nz = 24;
  lbmgpu_dist d{0, 1, -1, 3, nullptr, 1};  // 3 emulated slabs, peer transport
  Kernel ka(make_descriptor("aa-soa"), small, PaddingPolicy::automatic(), 0, &d);
  CHECK(throws<ConfigError>([&] { ka.peer_export(); }));
  lbmgpu_dist dp{0, 1, -1, 3, nullptr, 1};
  CHECK(throws<ConfigError>(
      [&] { Kernel kp(make_descriptor("list-aa-soa"), small, PaddingPolicy::automatic(), 0, &dp); }));
}

// verify_kernel (verification.cpp) through the C++ API
static void verification() {
  PoiseuilleCase c;
  c.nx = 4;
  c.ny = 4;
  c.nz = 18;
  const VerificationReport r = verify_kernel(make_descriptor("aa-soa"), c);
  CHECK(r.converged && r.passed && r.linf_rel < 1e-6);
}

// lbmgpu_run: one job equals load_state + advance + snapshot, bitwise, with
// page-locked buffers (pipelined schedule) and with pageable ones
static void run_job() {
  setenv("LBMGPU_FUSED_MB", "0", 1);  // small box: per-sweep launches, as for large lattices
  GeometrySpec ch;
  ch.kind = GeometryKind::Channel;
  ch.nx = 32;
  ch.ny = 16;
  ch.nz = 40;
  auto ref = make_kernel(make_descriptor("aa-soa"), ch);
  auto k = make_kernel(make_descriptor("aa-soa"), ch);
  ref->load_perturbed(77);
  const std::vector<double> init = ref->snapshot();
  ref->advance(kParams, kForce, 10);
  const std::vector<double> expect = ref->snapshot();
  const std::size_t n = init.size();
  void *pin_in = nullptr, *pin_out = nullptr;
  CHECK(lbmgpu_host_alloc(n * 8, &pin_in) == LBMGPU_OK);
  CHECK(lbmgpu_host_alloc(n * 8, &pin_out) == LBMGPU_OK);
  std::span<double> in(static_cast<double*>(pin_in), n), out(static_cast<double*>(pin_out), n);
  std::copy(init.begin(), init.end(), in.begin());
  CHECK(k->run(in, kParams, kForce, 10, out));  // pipelined
  CHECK(std::equal(out.begin(), out.end(), expect.begin()));
  auto k2 = make_kernel(make_descriptor("aa-soa"), ch);
  std::vector<double> out2(n);
  CHECK(!k2->run(init, kParams, kForce, 10, out2));  // pageable: the plain sequence
  CHECK(out2 == expect);
  CHECK(throws<ConfigError>([&] { k2->run(init, kParams, kForce, 3, out2); }));
  lbmgpu_host_free(pin_in);
  lbmgpu_host_free(pin_out);
  unsetenv("LBMGPU_FUSED_MB");
}

// perf-model arithmetic and the run coding (test_perfmodel.cpp:34-72,
// test_list_lattice.cpp:192-209) through the C++ wrappers
static void model_and_runs() {
  CHECK(std::fabs(loop_balance("list-aa-ria-soa", 3, 98).ref_min - 305.2) < 0.05);
  CHECK(loop_balance("list-aa-ria-soa", 0, 1000).ref_min == 304.0);
  CHECK(loop_balance("list-aa-ria-soa", 1000, 1000).ref_max == 342.0);
  const LoopBalance pull = loop_balance("list-pull-aos");
  CHECK(std::fabs(roofline(48.0, pull.ref_min, pull.ref_max).pmax_min_mflups - 90.909) < 0.1);
  CHECK(throws<ConfigError>([] { roofline(0.0, 304.0, 304.0); }));
  GeometrySpec g;
  g.kind = GeometryKind::Channel;
  g.nx = 20;
  g.ny = 10;
  g.nz = 10;
  Kernel ria(make_descriptor("list-aa-ria-soa"), g, PaddingPolicy::none());
  const std::vector<std::uint32_t> starts = ria.export_runs();
  CHECK(starts.size() == 3u * 20 * 8);  // (1, 6, 1) per z line of 8
  CHECK(starts.size() >= 3 && starts[0] == 0 && starts[1] == 1 && starts[2] == 7);
  CHECK(ria.vectorizable_fraction(4).value_or(-1) == 0.5);
  CHECK(ria.vectorizable_fraction(1).value_or(-1) == 1.0);
  Kernel plain(make_descriptor("list-aa-soa"), g, PaddingPolicy::none());
  CHECK(plain.export_runs().empty() && !plain.vectorizable_fraction(4).has_value());
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::printf("usage: cpp_api_test FULL_FP HALF_FP\n");
    return 2;
  }
  try {
    registry();
    fixed_point();
    golden(argv[1], argv[2]);
    rejections();
    verification();
    run_job();
    model_and_runs();
  } catch (const std::exception& e) {
    std::printf("unexpected exception: %s\n", e.what());
    return 1;
  }
  if (failures) {
    std::printf("%d FAILED\n", failures);
    return 1;
  }
  std::printf("ALL PASSED\n");
  return 0;
}

// Reference-side proof of the drop-in (VERDICT r1, next-round task 3): the
// unmodified lbmbench library (oracle/_ref/obj, built from
// /root/reference/proj/src) drives the GPU kernel through its own
// lbm::Kernel interface, next to its CPU make_kernel on the same FlagField:
//  * Kernel::advance -- the reference's base-class validation
//    (kernels.cpp:84-93): an odd AA count and a negative count throw
//    ConfigError and leave the GPU state untouched;
//  * lbm::state_fingerprint (harness.cpp:27-39) of the GPU snapshot equals
//    the CPU kernel's, and total_mass agrees to 1e-12;
//  * lbm::steady_state_run (harness.cpp:141-174) runs on the GPU kernel and
//    stops after the same step count as on the CPU kernel.
// Prints one PASS/FAIL line per case; exit code 0 iff all passed.
//   dropin_check [name ...]      (default: aa-soa blk-push-soa list-aa-soa list-pull-soa)
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "kernels_gpu.hpp"
#include "lbm/errors.hpp"
#include "lbm/geometry.hpp"
#include "lbm/harness.hpp"
#include "lbm/kernels.hpp"
#include "lbm/workers.hpp"

namespace {

using namespace lbm;

const TrtParams kParams = TrtParams::from_tau(0.9);  // tests/test_kernels.cpp:14-15
const BodyForce kForce{{1e-5, 2e-6, -3e-6}};

bool rejects_before_touching(Kernel& k, long steps) {
  const std::uint64_t before = state_fingerprint(k.snapshot());
  try {
    k.advance(kParams, kForce, steps);
    return false;
  } catch (const ConfigError&) {
  }
  return state_fingerprint(k.snapshot()) == before;
}

bool check(const std::string& name, const GeometrySpec& spec, const char* tag) {
  const FlagField ff = build_geometry(spec);
  const KernelDescriptor desc = make_descriptor(name);
  WorkerPool pool(2);
  std::unique_ptr<Kernel> cpu = make_kernel(desc, ff, PaddingPolicy::automatic(), pool);
  std::unique_ptr<Kernel> gpu = gpu::make_gpu_kernel(desc, ff, PaddingPolicy::automatic());
  Kernel& c = *cpu;
  Kernel& g = *gpu;
  bool ok = c.n_fluid() == g.n_fluid();
  const std::vector<double> init = perturbed_equilibrium(c.n_fluid(), 1234);
  c.load_state(init);
  g.load_state(init);
  ok = ok && rejects_before_touching(g, -2);
  if (desc.prop == Propagation::Aa) ok = ok && rejects_before_touching(g, 3);
  c.advance(kParams, kForce, 8);
  g.advance(kParams, kForce, 8);
  c.advance(kParams, kForce, 2);
  g.advance(kParams, kForce, 2);
  const std::uint64_t fc = state_fingerprint(c.snapshot());
  const std::uint64_t fg = state_fingerprint(g.snapshot());
  const double mc = c.total_mass(), mg = g.total_mass();
  ok = ok && fc == fg && std::fabs(mc - mg) <= 1e-12 * std::fabs(mc);
  // the reference's steady-state driver over both kernels
  const SteadyStateResult sc = steady_state_run(c, kParams, kForce, 20, 1e-3, 400);
  const SteadyStateResult sg = steady_state_run(g, kParams, kForce, 20, 1e-3, 400);
  const bool steady = sc.steps == sg.steps && sc.converged == sg.converged &&
                      state_fingerprint(c.snapshot()) == state_fingerprint(g.snapshot());
  ok = ok && steady;
  std::printf("%s %s %s %dx%dx%d n_fluid=%zu fingerprint cpu=%016llx gpu=%016llx "
              "steady_steps cpu=%ld gpu=%ld\n",
              ok ? "PASS" : "FAIL", name.c_str(), tag, spec.nx, spec.ny, spec.nz, g.n_fluid(),
              static_cast<unsigned long long>(fc), static_cast<unsigned long long>(fg), sc.steps,
              sg.steps);
  return ok;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> names;
  for (int i = 1; i < argc; ++i) names.emplace_back(argv[i]);
  if (names.empty()) names = {"aa-soa", "blk-push-soa", "list-aa-soa", "list-pull-soa"};
  bool all = true;
  try {
    for (const std::string& n : names) {
      all &= check(n, {GeometryKind::Blocks, 12, 10, 10, 4, 4}, "blocks");
      all &= check(n, {GeometryKind::Channel, 32, 12, 8, 4, 4}, "channel");
    }
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1;
  }
  return all ? 0 : 1;
}

// The drop-in binding a maintainer adds to lbmbench:
// an lbm::Kernel (reference proj/include/lbm/kernels.hpp:58-96) whose
// lattice and sweeps live on the B200, forwarding every virtual to the C ABI
// of include/lbmgpu.h.  Nothing here is copied from the reference: it only
// includes the reference's public headers.  Built against the unmodified
// reference objects by integration/Makefile; exercised by dropin_check.cpp.
#include "kernels_gpu.hpp"

#include <lbmgpu.h>

#include <string>
#include <utility>

namespace lbm::gpu {
namespace {

// lbmgpu status -> the reference's exception classes (errors.hpp:9-18); a
// device failure has no reference class and surfaces as runtime_error.
void gpu_check(int rc) {
  if (rc == LBMGPU_OK) return;
  const std::string msg = lbmgpu_last_error();
  if (rc == LBMGPU_ECONFIG) throw ConfigError(msg);
  if (rc == LBMGPU_ENUMERICAL) throw NumericalError(msg);
  throw std::runtime_error("lbmgpu device error: " + msg);
}

class GpuKernel final : public Kernel {
 public:
  GpuKernel(KernelDescriptor d, const FlagField& ff, const PaddingPolicy& pad, int row_pad)
      : Kernel(std::move(d)) {
    lbmgpu_geometry g{};
    g.kind = LBMGPU_CUSTOM;  // any FlagField (kernels.hpp:102-105)
    g.nx = ff.nx;
    g.ny = ff.ny;
    g.nz = ff.nz;
    g.flags = ff.flags.data();
    for (int a = 0; a < 3; ++a) g.periodic[a] = ff.periodic[a] ? 1 : 0;
    lbmgpu_padding p{};
    p.mode = static_cast<int>(pad.mode);  // None, Auto, Thrash, Explicit
    for (int q = 0; q < kQ; ++q) p.pads[q] = pad.pads[q];
    gpu_check(lbmgpu_create(desc_.name.c_str(), desc_.blk, desc_.vector_width, &g, &p, row_pad,
                            nullptr, &ctx_));
  }
  ~GpuKernel() override { lbmgpu_destroy(ctx_); }

  std::size_t n_fluid() const override {
    uint64_t n = 0;
    gpu_check(lbmgpu_n_fluid(ctx_, &n));
    return n;
  }
  KernelCaps capabilities() const override {
    int a = 0, b = 0, c = 0;
    gpu_check(lbmgpu_capabilities(ctx_, &a, &b, &c));
    return {a != 0, b, c != 0};
  }
  std::vector<double> snapshot() const override {
    std::vector<double> s(n_fluid() * kQ);
    gpu_check(lbmgpu_snapshot(ctx_, s.data(), s.size()));
    return s;
  }
  void load_state(std::span<const double> s) override {
    gpu_check(lbmgpu_load_state(ctx_, s.data(), s.size()));
  }
  double total_mass() const override {
    double m = 0;
    gpu_check(lbmgpu_total_mass(ctx_, &m));
    return m;
  }
  std::optional<RiaStats> ria_stats() const override {
    int64_t r = 0, n = 0;
    double v = 0, pv = 0;
    gpu_check(lbmgpu_ria_stats(ctx_, &r, &n, &v, &pv));
    if (r < 0) return std::nullopt;
    return RiaStats{static_cast<std::size_t>(r), static_cast<std::size_t>(n)};
  }

 protected:
  // Kernel::advance (kernels.cpp:84-93) has validated the arguments and
  // rejected odd AA counts before this is reached.
  void do_advance(const TrtParams& p, const BodyForce& g, long steps) override {
    gpu_check(lbmgpu_advance(ctx_, p.omega_plus, p.magic_lambda, g.g.data(), steps));
  }

 private:
  lbmgpu_ctx* ctx_ = nullptr;
};

}  // namespace

std::unique_ptr<Kernel> make_gpu_kernel(const KernelDescriptor& d, const FlagField& ff,
                                        const PaddingPolicy& pad, int row_pad) {
  return std::make_unique<GpuKernel>(d, ff, pad, row_pad);
}

}  // namespace lbm::gpu

// D3Q19 TRT collision with simple body forcing, in registers.
//
// Restates collide_node (reference include/lbm/d3q19.hpp:107-144) with the
// SAME expression trees and evaluation order; the library is compiled with
// --fmad=false (device) and -ffp-contract=off (host), the reference with
// -ffp-contract=off (CMakeLists.txt:12-14), so every rounding step is the
// reference's and results are bit-identical.  The only restructuring is that
// c_i.g (a per-direction constant) is evaluated once on the host with the
// reference's expression and passed in (TrtArgs::cg); this is exact.
#pragma once

#include "common.cuh"

namespace lbmgpu {

struct TrtArgs {
  double wp;      // omega_plus
  double wm;      // omega_minus (d3q19.hpp:70-73, evaluated on the host)
  double cg[kQ];  // cg[i] = c_i.g for the odd i of each (i, i+1) pair
};

// Host-side construction.  The expression for cg is d3q19.hpp:132.
inline TrtArgs make_trt(double omega_plus, double omega_minus,
                        const double* g) {
  TrtArgs t{};
  t.wp = omega_plus;
  t.wm = omega_minus;
  for (int i = 0; i < kQ; ++i)
    t.cg[i] = static_cast<double>(cx(i)) * g[0] +
              static_cast<double>(cy(i)) * g[1] +
              static_cast<double>(cz(i)) * g[2];
  return t;
}

// d3q19.hpp:70-73
inline double omega_minus_of(double omega_plus, double magic_lambda) {
  const double kappa = 1.0 / omega_plus - 0.5;
  return 1.0 / (0.5 + magic_lambda / kappa);
}

template <int I>
__device__ __forceinline__ double cdot(double ux, double uy, double uz) {
  // kC[i][0]*ux + kC[i][1]*uy + kC[i][2]*uz with the integer stencil entry
  // converted to double, exactly as the reference's int*double products.
  // Products by +-1 are exact and may be folded by the compiler; products by
  // 0 are kept (IEEE: 0*x is not foldable without fast-math).
  return static_cast<double>(cx(I)) * ux + static_cast<double>(cy(I)) * uy +
         static_cast<double>(cz(I)) * uz;
}

template <int I>
__device__ __forceinline__ void relax_pair(double (&f)[kQ], double rho,
                                           double ux, double uy, double uz,
                                           double one_m, const TrtArgs& a) {
  constexpr int J = I + 1;
  const double cu = cdot<I>(ux, uy, uz);
  const double wr = weight(I) * rho;
  const double e_even = wr * (one_m + 4.5 * cu * cu);
  const double e_odd = wr * 3.0 * cu;
  const double f_even = 0.5 * (f[I] + f[J]);
  const double f_odd = 0.5 * (f[I] - f[J]);
  const double d_even = a.wp * (f_even - e_even);
  const double d_odd = a.wm * (f_odd - e_odd);
  const double forcing = wr * 3.0 * a.cg[I];
  f[I] = f[I] - d_even - d_odd + forcing;
  f[J] = f[J] - d_even + d_odd - forcing;
}

__device__ __forceinline__ void collide(double (&f)[kQ], const TrtArgs& a) {
  double rho = f[0];
#pragma unroll
  for (int i = 1; i < kQ; ++i) rho += f[i];
  const double mx = f[1] - f[2] + f[7] - f[8] + f[9] - f[10] + f[11] - f[12] +
                    f[13] - f[14];
  const double my = f[3] - f[4] + f[7] - f[8] - f[9] + f[10] + f[15] - f[16] +
                    f[17] - f[18];
  const double mz = f[5] - f[6] + f[11] - f[12] - f[13] + f[14] + f[15] -
                    f[16] - f[17] + f[18];
  const double inv_rho = 1.0 / rho;
  const double ux = mx * inv_rho;
  const double uy = my * inv_rho;
  const double uz = mz * inv_rho;
  const double usq = ux * ux + uy * uy + uz * uz;
  const double one_m = 1.0 - 1.5 * usq;
  f[0] -= a.wp * (f[0] - kWRest * rho * one_m);
  relax_pair<1>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<3>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<5>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<7>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<9>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<11>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<13>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<15>(f, rho, ux, uy, uz, one_m, a);
  relax_pair<17>(f, rho, ux, uy, uz, one_m, a);
}

// Bare moments (reference src/d3q19.cpp:20-34): rho = sum f,
// u = (sum c f) / rho, accumulated in direction order.
__device__ __forceinline__ void macroscopic(const double (&f)[kQ], double& rho,
                                            double& ux, double& uy,
                                            double& uz) {
  double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
  for (int i = 0; i < kQ; ++i) {
    r += f[i];
    mx += static_cast<double>(cx(i)) * f[i];
    my += static_cast<double>(cy(i)) * f[i];
    mz += static_cast<double>(cz(i)) * f[i];
  }
  rho = r;
  ux = mx / r;
  uy = my / r;
  uz = mz / r;
}

}  // namespace lbmgpu

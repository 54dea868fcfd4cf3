// Standalone experiment (not part of the library): where does the AA odd
// sub-step lose bandwidth against the even one?  Runs the odd access pattern
// with parts of the neighbour shift switched off on a cfg-5-shaped lattice
// (channel 1024 x 512 x NZ, [z][slot][y][x] SoA) and prints GB/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false \
//        -I../paper_1711_11468_b200/csrc -o aa_odd_experiments aa_odd_experiments.cu
#include <cstdio>
#include <vector>

#include "model.cuh"

using namespace lbmgpu;

struct A {
  double* buf;
  uint32_t nx, ny, nz;
  uint64_t P;
  TrtArgs trt;
};

// SX/SY/SZ: apply the x/y/z neighbour shift on loads (L) and stores (S)
template <bool LX, bool LYZ, bool SX, bool SYZ, bool COLL>
__global__ void __launch_bounds__(256, 2) k_var(const A a) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t P = static_cast<uint32_t>(a.P);
  const uint32_t z = n / P, r = n - z * P, y = r / a.nx, x = r - y * a.nx;
  if (z == 0 || z + 1 >= a.nz || y == 0 || y + 1 >= a.ny) return;  // channel walls
  const uint32_t X[3] = {x == 0 ? a.nx - 1 : x - 1, x, x + 1 == a.nx ? 0 : x + 1};
  auto idx = [&](uint32_t zz, int s, uint32_t yy, uint32_t xx) {
    return (uint64_t(zz) * kQ + s) * a.P + uint64_t(yy) * a.nx + xx;
  };
  double q[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) {
    const uint32_t zz = LYZ ? z - cz(d) : z, yy = LYZ ? y - cy(d) : y;
    const uint32_t xx = LX ? X[1 - cx(d)] : x;
    q[d] = a.buf[idx(zz, dslot(opp(d)), yy, xx)];
  }
  if (COLL) collide(q, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d) {
    const uint32_t zz = SYZ ? z + cz(d) : z, yy = SYZ ? y + cy(d) : y;
    const uint32_t xx = SX ? X[1 + cx(d)] : x;
    a.buf[idx(zz, dslot(d), yy, xx)] = q[d];
  }
}

// even step with two x-adjacent nodes per thread and 16-byte accesses
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_even_vec2(const A a) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t P = static_cast<uint32_t>(a.P);
  const uint32_t n = 2 * t;
  const uint32_t z = n / P, r = n - z * P, y = r / a.nx, x = r - y * a.nx;
  if (z == 0 || z + 1 >= a.nz || y == 0 || y + 1 >= a.ny) return;
  const uint64_t base = (uint64_t(z) * kQ) * a.P + uint64_t(y) * a.nx + x;
  double q0[kQ], q1[kQ];
#pragma unroll
  for (int d = 0; d < kQ; ++d) {
    const double2 v = *reinterpret_cast<const double2*>(a.buf + base + uint64_t(dslot(d)) * a.P);
    q0[d] = v.x;
    q1[d] = v.y;
  }
  collide(q0, a.trt);
  collide(q1, a.trt);
#pragma unroll
  for (int d = 0; d < kQ; ++d)
    *reinterpret_cast<double2*>(a.buf + base + uint64_t(dslot(opp(d))) * a.P) =
        make_double2(q0[d], q1[d]);
}

template <class K>
double timeit2(K k, const A& a, uint64_t nodes, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned grid = static_cast<unsigned>((nodes / 2 + 255) / 256);
  k<<<grid, 256>>>(a);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<grid, 256>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fluid = double(a.nx) * (a.ny - 2) * (a.nz - 2);
  return fluid * 304.0 * reps / (ms / 1e3) / 1e9;
}

template <class K>
double timeit(K k, const A& a, uint64_t nodes, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned grid = static_cast<unsigned>((nodes + 255) / 256);
  k<<<grid, 256>>>(a);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<grid, 256>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fluid = double(a.nx) * (a.ny - 2) * (a.nz - 2);
  return fluid * 304.0 * reps / (ms / 1e3) / 1e9;
}

int main(int argc, char** argv) {
  const uint32_t nx = 1024, ny = 512, nz = argc > 1 ? atoi(argv[1]) : 256;
  A a;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.P = uint64_t(nx) * ny;
  const double g[3] = {1e-5, 0, 0};
  a.trt = make_trt(1.0, omega_minus_of(1.0, 3.0 / 16.0), g);
  const uint64_t nodes = a.P * nz;
  cudaMalloc(&a.buf, nodes * kQ * 8);
  std::vector<double> w(kQ);
  {
    std::vector<double> h(a.P);
    for (int s = 0; s < kQ; ++s) {
      for (auto& v : h) v = weight(ddir(s));
      for (uint32_t z = 0; z < nz; ++z)
        cudaMemcpy(a.buf + (uint64_t(z) * kQ + s) * a.P, h.data(), a.P * 8, cudaMemcpyHostToDevice);
    }
  }
  const int reps = 10;
  printf("nz=%u fluid=%.0f (GB/s at 304 B/node)\n", nz, double(nx) * (ny - 2) * (nz - 2));
  printf("even-like (no shift)         %8.1f\n", timeit(k_var<false, false, false, false, true>, a, nodes, reps));
  printf("odd (all shifts)             %8.1f\n", timeit(k_var<true, true, true, true, true>, a, nodes, reps));
  printf("x shift only (ld+st)         %8.1f\n", timeit(k_var<true, false, true, false, true>, a, nodes, reps));
  printf("y/z shift only (ld+st)       %8.1f\n", timeit(k_var<false, true, false, true, true>, a, nodes, reps));
  printf("shifted loads, local stores  %8.1f\n", timeit(k_var<true, true, false, false, true>, a, nodes, reps));
  printf("local loads, shifted stores  %8.1f\n", timeit(k_var<false, false, true, true, true>, a, nodes, reps));
  printf("odd, no collide              %8.1f\n", timeit(k_var<true, true, true, true, false>, a, nodes, reps));
  printf("even, no collide             %8.1f\n", timeit(k_var<false, false, false, false, false>, a, nodes, reps));
  printf("even vec2 (2 nodes/thr) mb1  %8.1f\n", timeit2(k_even_vec2<1>, a, nodes, reps));
  printf("even vec2 (2 nodes/thr) mb2  %8.1f\n", timeit2(k_even_vec2<2>, a, nodes, reps));
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}

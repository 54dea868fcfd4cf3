// Zero-copy (SM-driven) PCIe bandwidth vs the copy engines on this box:
// coalesced 16-byte loads from / stores to mapped pinned host memory by a
// small grid, alone and beside an HBM-bound kernel on another stream.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void zc_read(const double2* __restrict__ h, double2* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) d[i] = h[i];
}
__global__ void zc_write(const double2* __restrict__ d, double2* __restrict__ h, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) h[i] = d[i];
}
__global__ void hbm_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) b[i] = a[i];
}
int main() {
  const size_t bytes = size_t(4) << 30, n = bytes / 16;
  double2 *h, *d, *a, *b;
  CK(cudaMallocHost(&h, bytes));
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  cudaMemset(d, 0, bytes); cudaMemset(a, 0, bytes);
  for (size_t i = 0; i < n; i += 4096) h[i] = make_double2(1, 2);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t e0, e1, f0, f1; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&f0); cudaEventCreate(&f1);
  float ms;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(e0, s1); cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("copy engine h2d %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(e0, s1); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("copy engine d2h %.1f GB/s\n", bytes / ms / 1e6);
  }
  for (int grid : {16, 32, 64, 148, 296}) {
    cudaEventRecord(e0, s1); zc_read<<<grid, 256, 0, s1>>>(h, d, n); cudaEventRecord(e1, s1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("zero-copy read  grid %3d: %.1f GB/s\n", grid, bytes / ms / 1e6);
    cudaEventRecord(e0, s1); zc_write<<<grid, 256, 0, s1>>>(d, h, n); cudaEventRecord(e1, s1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("zero-copy write grid %3d: %.1f GB/s\n", grid, bytes / ms / 1e6);
  }
  // alone: HBM copy
  cudaEventRecord(f0, s2); hbm_copy<<<148 * 8, 256, 0, s2>>>(a, b, n, 20); cudaEventRecord(f1, s2); CK(cudaEventSynchronize(f1));
  cudaEventElapsedTime(&ms, f0, f1); printf("hbm copy alone %.0f GB/s\n", 2.0 * bytes * 20 / ms / 1e6);
  for (int grid : {32, 64}) {
    for (int dir = 0; dir < 3; ++dir) {
      cudaEventRecord(f0, s2); hbm_copy<<<148 * 8, 256, 0, s2>>>(a, b, n, 20); cudaEventRecord(f1, s2);
      cudaEventRecord(e0, s1);
      if (dir == 0) zc_read<<<grid, 256, 0, s1>>>(h, d, n);
      else if (dir == 1) zc_write<<<grid, 256, 0, s1>>>(d, h, n);
      else cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1);
      cudaEventRecord(e1, s1);
      CK(cudaEventSynchronize(f1)); CK(cudaEventSynchronize(e1));
      float ms2; cudaEventElapsedTime(&ms, f0, f1); cudaEventElapsedTime(&ms2, e0, e1);
      printf("concurrent (%s grid %d): hbm copy %.0f GB/s, transfer %.1f GB/s\n", dir == 0 ? "zc read" : dir == 1 ? "zc write" : "copy engine h2d", grid, 2.0 * bytes * 20 / ms / 1e6, bytes / ms2 / 1e6);
    }
  }
  return 0;
}

// cudaMemcpy2DAsync throughput (pinned host <-> device) for the row widths a
// z-slab of the cfg-5 channel has in the reference's x-major canonical order:
// rows of (nz - 2) * 152 B, slab segments of w planes * 152 B.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t pitch = 510 * 152, rows = 1024 * 510;  // cfg 5: nz-2 = 510 fluid z, nx * (ny-2) rows
  const size_t hbytes = pitch * rows;                  // 40.5 GB
  char *h, *d;
  if (cudaMallocHost(&h, hbytes) != cudaSuccess) { printf("host alloc failed\n"); return 1; }
  if (cudaMalloc(&d, size_t(64) * 152 * rows) != cudaSuccess) { printf("dev alloc failed\n"); return 1; }
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {2, 4, 8, 16, 32, 64}) {
    const size_t width = size_t(w) * 152;
    for (int dir = 0; dir < 2; ++dir) {
      float best = 1e9;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0, s);
        if (dir == 0) cudaMemcpy2DAsync(d, width, h + 152 * 100, pitch, width, rows, cudaMemcpyHostToDevice, s);
        else cudaMemcpy2DAsync(h + 152 * 100, pitch, d, width, width, rows, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("2D %s width %5zu B (%2d planes): %.1f GB/s (%.1f ms)\n", dir ? "d2h" : "h2d", width, w, width * rows / best / 1e6, best);
    }
  }
  printf("error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

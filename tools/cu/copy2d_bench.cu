// Pinned H2D/D2H bandwidth: contiguous vs 2D pitched copies of a 5760-row
// chunk of 92162 fp32 columns, each direction alone and both at once.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
int main() {
  const size_t cols = 92162, rows = 5760, w = cols * 4, pitch = ((cols + 31) / 32 * 32) * 4;
  const size_t bytes = rows * w;
  char *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, bytes, 0); cudaHostAlloc(&h2, bytes, 0);
  cudaMalloc(&d1, rows * pitch); cudaMalloc(&d2, rows * pitch);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, int mode, bool twod) {
    float best = 1e9;
    for (int it = 0; it < 4; ++it) {
      cudaDeviceSynchronize(); cudaEventRecord(a, 0);
      cudaStreamWaitEvent(s1, a); cudaStreamWaitEvent(s2, a);
      if (mode & 1) { if (twod) cudaMemcpy2DAsync(d1, pitch, h1, w, w, rows, cudaMemcpyHostToDevice, s1);
                      else cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1); }
      if (mode & 2) { if (twod) cudaMemcpy2DAsync(h2, w, d2, pitch, w, rows, cudaMemcpyDeviceToHost, s2);
                      else cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2); }
      cudaEvent_t e1, e2; cudaEventCreate(&e1); cudaEventCreate(&e2);
      cudaEventRecord(e1, s1); cudaEventRecord(e2, s2); cudaStreamWaitEvent(0, e1); cudaStreamWaitEvent(0, e2);
      cudaEventRecord(b, 0); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-24s %s  %.2f ms  %.1f GB/s per direction\n", name, twod ? "2D" : "1D", best, bytes / best / 1e6);
  };
  for (int twod = 0; twod < 2; ++twod) { run("h2d", 1, twod); run("d2h", 2, twod); run("duplex", 3, twod); }
  return 0;
}

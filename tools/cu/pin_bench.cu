// Duplex H2D+D2H bandwidth vs host allocation kind: cudaHostAlloc,
// malloc+cudaHostRegister, mmap(MADV_HUGEPAGE)+cudaHostRegister.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
int main() {
  const size_t bytes = size_t(2) << 30;
  char *d1, *d2;
  cudaMalloc(&d1, bytes); cudaMalloc(&d2, bytes);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b, e1, e2; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&e1); cudaEventCreate(&e2);
  for (int kind = 0; kind < 3; ++kind) {
    char *h1, *h2;
    if (kind == 0) { cudaHostAlloc(&h1, bytes, 0); cudaHostAlloc(&h2, bytes, 0); }
    else if (kind == 1) { h1 = (char*)malloc(bytes); h2 = (char*)malloc(bytes); memset(h1, 1, bytes); memset(h2, 1, bytes);
      cudaHostRegister(h1, bytes, 0); cudaHostRegister(h2, bytes, 0); }
    else { h1 = (char*)mmap(0, bytes, PROT_READ|PROT_WRITE, MAP_PRIVATE|MAP_ANONYMOUS, -1, 0);
      h2 = (char*)mmap(0, bytes, PROT_READ|PROT_WRITE, MAP_PRIVATE|MAP_ANONYMOUS, -1, 0);
      madvise(h1, bytes, MADV_HUGEPAGE); madvise(h2, bytes, MADV_HUGEPAGE); memset(h1, 1, bytes); memset(h2, 1, bytes);
      cudaHostRegister(h1, bytes, 0); cudaHostRegister(h2, bytes, 0); }
    for (int mode = 1; mode <= 3; ++mode) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        cudaDeviceSynchronize(); cudaEventRecord(a, 0); cudaStreamWaitEvent(s1, a); cudaStreamWaitEvent(s2, a);
        if (mode & 1) cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
        if (mode & 2) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e1, s1); cudaEventRecord(e2, s2); cudaStreamWaitEvent(0, e1); cudaStreamWaitEvent(0, e2);
        cudaEventRecord(b, 0); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("%s %-7s %.1f GB/s per direction\n", kind == 0 ? "hostalloc   " : kind == 1 ? "malloc+reg  " : "hugepage+reg",
             mode == 1 ? "h2d" : mode == 2 ? "d2h" : "duplex", bytes / best / 1e6);
    }
  }
  return 0;
}

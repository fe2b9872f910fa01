// FP32 FMA-pipe peak on this B200: FFMA2 (fma.rn.f32x2) vs scalar FFMA, with the
// multiplier in a uniform register (the K1 weight form) and 8 independent chains
// per thread. Prints TFMA/s (fused multiply-adds per second, each counting 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

template <int CH>
__global__ void k_ffma2(float w, int iters, float* out) {
  uint64_t acc[CH];
  const float t = threadIdx.x * 1e-7f;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = pk(t + c, t - c);
  const uint64_t ww = pk(w, w);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(acc[c]) : "l"(ww), "l"(ww));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(acc[c]));
    s += a + b;
  }
  if (s == 12345.f) out[0] = s;
}

template <int CH>
__global__ void k_ffma(float w, int iters, float* out) {
  float acc[CH];
  const float t = threadIdx.x * 1e-7f;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = t + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32 %0, %1, %0, %1;" : "+f"(acc[c]) : "f"(w));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int nt : {256, 512, 1024}) {
    for (int pass = 0; pass < 2; ++pass) {
      float ms;
      const int blocks = sms * (2048 / nt);
      cudaEventRecord(a);
      k_ffma2<8><<<blocks, nt>>>(1.0000001f, iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      const double f2 = double(blocks) * nt * iters * 8 * 2 / (ms * 1e-3) / 1e12;
      cudaEventRecord(a);
      k_ffma<16><<<blocks, nt>>>(1.0000001f, iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      const double f1 = double(blocks) * nt * iters * 16 / (ms * 1e-3) / 1e12;
      if (pass) printf("{\"threads_per_cta\": %d, \"ffma2_TFMAps\": %.2f, \"ffma_TFMAps\": %.2f}\n", nt, f2, f1);
    }
  }
  // one warp per SMSP (latency-bound ILP test): 4 warps per SM
  for (int pass = 0; pass < 2; ++pass) {
    float ms;
    cudaEventRecord(a);
    k_ffma2<8><<<sms, 128>>>(1.0000001f, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass)
      printf("{\"warps_per_smsp\": 1, \"ffma2_TFMAps\": %.2f}\n", double(sms) * 128 * iters * 16 / (ms * 1e-3) / 1e12);
  }
  return 0;
}

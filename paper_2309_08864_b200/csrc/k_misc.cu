// k_misc.cu -- K1 dispatch and the small device kernels:
//   K6 synthetic init (splitmix64, bit-identical to proj/src/stencil.cpp:91-118).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <unordered_map>

#include "k1_launch.h"

namespace so2dr_dev {

int device_sm_count() {
  static std::atomic<int> cached[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int n = cached[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int k1_max_steps(int dim, int dtype, int kind, int radius) {
  if (dim == 2) {
    if (kind == KGRAD) return radius == 1 ? 8 : 0;
    if (radius < 1 || radius > 4) return 0;
    // must match maxs2d() in k1_2d_impl.cuh
    if (dtype == 0) return radius == 1 ? 8 : 4;
    return radius == 1 ? 8 : radius == 2 ? 4 : radius == 3 ? 2 : 1;
  }
  if (dim == 3) {
    if (kind == KGRAD) return 0;
    if (radius < 1 || radius > 2) return 0;
    // must match maxs3d() in k1_3d.cu
    if (dtype == 0) return radius == 1 ? 4 : 2;
    return radius == 1 ? 2 : 1;
  }
  return 0;
}

cudaError_t k1_launch(const K1Launch& L, cudaStream_t stream) {
  if (L.dim == 2) return L.dtype == 0 ? launch_k1_2d_f32(L, stream) : launch_k1_2d_f64(L, stream);
  if (L.dim == 3) return L.dtype == 0 ? launch_k1_3d_f32(L, stream) : launch_k1_3d_f64(L, stream);
  return cudaErrorInvalidValue;
}

uint64_t k1_alg_bytes(const K1Launch& L) {
  const int top_in = std::min(L.base + L.rows, L.y1 + L.radius * L.steps);
  const int bot_in = std::max(L.base, L.y0 - L.radius * L.steps);
  const uint64_t unit = static_cast<uint64_t>(L.dim == 3 ? (int64_t)L.plane_rows * L.cols : L.cols) *
                        (L.dtype == 1 ? 8 : 4);
  return static_cast<uint64_t>((top_in - bot_in) + (L.y1 - L.y0)) * unit;
}

// ---- K6: synthetic init ----------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void init_kernel(T* out, int64_t pitch, int p, int dim, int64_t lo, int64_t n_units,
                            uint64_t seed) {
  // one thread per cell of units [lo, lo + n_units); unit = row (2D) / plane (3D)
  const int64_t rows_per_unit = dim == 3 ? p : 1;
  const int64_t total_rows = n_units * rows_per_unit;
  for (int64_t row = blockIdx.y; row < total_rows; row += gridDim.y) {
    const int64_t unit = lo + row / rows_per_unit;
    const int y = dim == 3 ? static_cast<int>(row % rows_per_unit) : static_cast<int>(unit);
    const uint64_t s = dim == 3 ? seed ^ (static_cast<uint64_t>(static_cast<uint32_t>(unit)) *
                                          0x9E3779B97F4A7C15ULL)
                                : seed;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < p; x += gridDim.x * blockDim.x) {
      const uint64_t key = (static_cast<uint64_t>(static_cast<uint32_t>(y)) << 32) |
                           static_cast<uint32_t>(x);
      const float v = static_cast<float>(mix64(s ^ mix64(key)) >> 40) * 0x1p-24f;
      out[row * pitch + x] = static_cast<T>(v);
    }
  }
}

cudaError_t launch_init(int dtype, void* out, int64_t pitch, int p, int dim, int64_t lo,
                        int64_t n_units, uint64_t seed, cudaStream_t stream) {
  const int64_t rows = n_units * (dim == 3 ? p : 1);
  dim3 block(256);
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((p + 255) / 256, 64)),
            static_cast<unsigned>(std::min<int64_t>(rows, 65535)));
  if (rows <= 0) return cudaSuccess;
  if (dtype == 0)
    init_kernel<float><<<grid, block, 0, stream>>>(static_cast<float*>(out), pitch, p, dim, lo,
                                                   n_units, seed);
  else
    init_kernel<double><<<grid, block, 0, stream>>>(static_cast<double*>(out), pitch, p, dim, lo,
                                                    n_units, seed);
  return cudaGetLastError();
}

}  // namespace so2dr_dev

// ---- work counters for the persistent K1 kernels ---------------------------
// One counter pair per (device, stream): [0] hands out work items, [1] counts
// the warps that left. The last warp of a launch re-arms both (k1_stencil2d),
// so launches on one stream -- which never overlap -- reuse the pair without
// a per-launch memset. Device globals start zeroed at module load.
namespace so2dr_dev {
constexpr unsigned kCounterPairs = 4096;
__device__ unsigned g_k1_counters[2 * kCounterPairs];

unsigned* k1_next_counter(cudaStream_t stream) {
  static std::mutex mu;
  static unsigned* base[64] = {};
  static std::unordered_map<uint64_t, unsigned> slots;
  static unsigned used[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_k1_counters) != cudaSuccess) return nullptr;
    base[dev] = static_cast<unsigned*>(p);
  }
  const uint64_t key = (static_cast<uint64_t>(dev) << 56) ^ reinterpret_cast<uintptr_t>(stream);
  auto it = slots.find(key);
  if (it == slots.end()) {
    if (used[dev] >= kCounterPairs) return nullptr;  // more live streams than pairs
    it = slots.emplace(key, used[dev]++).first;
  }
  return base[dev] + 2 * it->second;
}
}  // namespace so2dr_dev

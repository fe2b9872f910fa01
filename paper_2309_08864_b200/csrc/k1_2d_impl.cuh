// k1_2d_impl.cuh -- launch-side dispatch of the 2D K1 kernels (included by
// k1_2d_f32.cu / k1_2d_f64.cu so the two element types compile in parallel).
#pragma once

#include <algorithm>
#include <cstring>
#include <utility>

#include "k1_2d.cuh"
#include "k1_launch.h"

namespace so2dr_dev {

constexpr int kThreads2D = 256;

template <typename T>
constexpr int v2d(int R) {
  return sizeof(T) == 4 ? 4 : (R <= 2 ? 2 : 4);
}
template <typename T>
constexpr int maxs2d(int R) {
  return sizeof(T) == 4 ? (R == 1 ? 8 : R == 2 ? 6 : 4) : (R == 1 ? 8 : R == 2 ? 6 : 2);
}

inline int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

template <typename T, int R, int S, int KIND>
cudaError_t launch_2d_fixed(const K1Launch& L, cudaStream_t stream) {
  constexpr int V = v2d<T>(R);
  constexpr int NT = kThreads2D;
  constexpr int H = R * S;
  constexpr int VEC = 16 / (int)sizeof(T);
  K1Args2D<T> a;
  a.in = static_cast<const T*>(L.in);
  a.out = static_cast<T*>(L.out);
  a.pitch = L.pitch;
  a.base = L.base;
  a.rows = L.rows;
  a.cols = L.cols;
  a.y0 = L.y0, a.y1 = L.y1, a.x0 = L.x0, a.x1 = L.x1;
  a.iy0 = L.iy0, a.iy1 = L.iy1, a.ix0 = L.ix0, a.ix1 = L.ix1;
  constexpr int E = 2 * R + 1;
  for (int i = 0; i < 81; ++i) a.w[i] = T(0);
  if (L.w)
    for (int i = 0; i < E * E; ++i) a.w[i] = static_cast<T>(L.w[i]);
  a.strip = ((NT * V - 2 * H) / VEC) * VEC;
  if (a.strip <= 0) return cudaErrorInvalidValue;
  a.xorg = floor_div(L.x0 - H, VEC) * VEC;
  const int width = L.x1 - (a.xorg + H);
  const int nx = std::max(1, (width + a.strip - 1) / a.strip);
  const int height = L.y1 - L.y0;
  // y segments: enough CTAs for ~4 waves at one CTA per SM, but keep each
  // segment long against its R*S warm-up + S*(R+1) pipeline fill.
  const int sms = device_sm_count();
  const int min_seg = std::max(48, 6 * (H + S * (R + 1)));
  const int max_ny = std::max(1, height / min_seg);
  int ny = std::max(1, (4 * sms + nx - 1) / nx);
  ny = std::min(ny, max_ny);
  a.seg = (height + ny - 1) / ny;
  ny = (height + a.seg - 1) / a.seg;
  dim3 grid(nx, ny);
  k1_stencil2d<T, R, S, KIND, V, NT><<<grid, NT, 0, stream>>>(a);
  return cudaGetLastError();
}

template <typename T, int R, int KIND, int S = 1>
cudaError_t launch_2d_s(const K1Launch& L, cudaStream_t stream) {
  if constexpr (S > maxs2d<T>(R)) {
    return cudaErrorInvalidValue;
  } else {
    if (L.steps == S) return launch_2d_fixed<T, R, S, KIND>(L, stream);
    return launch_2d_s<T, R, KIND, S + 1>(L, stream);
  }
}

template <typename T>
cudaError_t launch_2d(const K1Launch& L, cudaStream_t stream) {
  if (L.steps < 1) return cudaErrorInvalidValue;
  switch (L.kind) {
    case KGRAD:
      if (L.radius != 1) return cudaErrorInvalidValue;
      return launch_2d_s<T, 1, KGRAD>(L, stream);
    case KBOX:
      switch (L.radius) {
        case 1: return launch_2d_s<T, 1, KBOX>(L, stream);
        case 2: return launch_2d_s<T, 2, KBOX>(L, stream);
        case 3: return launch_2d_s<T, 3, KBOX>(L, stream);
        case 4: return launch_2d_s<T, 4, KBOX>(L, stream);
      }
      break;
    case KSTAR:
      switch (L.radius) {
        case 1: return launch_2d_s<T, 1, KSTAR>(L, stream);
        case 2: return launch_2d_s<T, 2, KSTAR>(L, stream);
        case 3: return launch_2d_s<T, 3, KSTAR>(L, stream);
        case 4: return launch_2d_s<T, 4, KSTAR>(L, stream);
      }
      break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace so2dr_dev

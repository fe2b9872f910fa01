// k1_2d_impl.cuh -- launch-side dispatch of the 2D K1 kernels (included by the
// k1_2d_{f32,f64}_r*.cu units so every (type, radius) compiles in parallel).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "k1_2d.cuh"
#include "k1_launch.h"
#include "k1_segplan.h"

namespace so2dr_dev {

constexpr int kThreads2D = 128;
#ifndef SO2DR_K1_MINB
#define SO2DR_K1_MINB 0
#endif

// cells per thread (V): 16 bytes per lane for r <= 2 (one cp.async / vector
// store per row), 4 cells for the wider fp64 radii (R <= V for the shuffles)
template <typename T>
constexpr int v2d(int R) {
  return sizeof(T) == 4 ? 4 : (R <= 2 ? 2 : 4);
}
// Steps fused per launch: S stages x the live accumulator rows must fit the
// register file without spilling (checked by test_no_kernel_uses_local_memory).
// Must match k1_max_steps() in k_misc.cu.
template <typename T>
constexpr int maxs2d(int R) {
  return sizeof(T) == 4 ? (R == 1 ? 8 : 4) : (R == 1 ? 8 : R == 2 ? 4 : R == 3 ? 2 : 1);
}

// resident 128-thread CTAs requested per SM (register cap 65536 / (128 minb)):
// the fused FMA pipeline needs enough warps to cover its fixed-latency chains
// (4 CTAs at S = 4 caps the kernel at 128 registers and spills; experiment
// builds set SO2DR_K1_MINB, tools/build_variant.sh)
// Larger radii / fp64 carry more accumulator rows: no cap (ptxas decides).
template <typename T>
constexpr int minb2d(int R, int S) {
  if (SO2DR_K1_MINB > 0) return SO2DR_K1_MINB;
  if (sizeof(T) == 4 && R == 1) return S <= 2 ? 4 : S <= 4 ? 3 : 2;
  return 1;
}

inline int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Work items per resident warp (row segments x strips) of the uniform
// segmentation, which also caps the guided plan's segment length
// (SO2DR_K1_IPW=n: experiments).
inline int k1_items_per_warp_override() {
  static int v = [] {
    const char* s = std::getenv("SO2DR_K1_IPW");
    return s ? std::max(1, std::atoi(s)) : 0;
  }();
  return v;
}
// SO2DR_K1_SEGS=uniform: the r02-mid uniform segmentation (A/B experiments)
inline bool k1_uniform_segments() {
  static bool v = [] {
    const char* s = std::getenv("SO2DR_K1_SEGS");
    return s && std::strcmp(s, "uniform") == 0;
  }();
  return v;
}

template <typename T, int R, int S, int KIND, int V>
cudaError_t launch_2d_fixed(const K1Launch& L, cudaStream_t stream) {
  constexpr int NT = kThreads2D;
  constexpr int H = R * S;
  using P = K1Plan2D<T, R, S, KIND, V, NT>;
  constexpr int VEC = P::VEC;
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
  for (int i = 0; i < 20; ++i) a.wp[i] = 0;
  if constexpr (std::is_same_v<T, float> && R <= 2) {
    for (int d = 1 - R; d <= R; ++d)
      for (int dx = -R; dx <= R; ++dx) {
        const float lo = a.w[(d + R) * E + dx + R], hi = a.w[(d - 1 + R) * E + dx + R];
        uint32_t bl, bh;
        std::memcpy(&bl, &lo, 4);
        std::memcpy(&bh, &hi, 4);
        a.wp[(d + R - 1) * E + dx + R] = (static_cast<uint64_t>(bh) << 32) | bl;
      }
  }
  {
    const int64_t pb = L.pitch * static_cast<int64_t>(sizeof(T));
    a.cpb = pb % 16 == 0 ? 16 : pb % 8 == 0 ? 8 : 4;
    a.aligned8 = pb % 8 == 0 && reinterpret_cast<uintptr_t>(L.in) % 8 == 0 &&
                 reinterpret_cast<uintptr_t>(L.out) % 8 == 0;
  }
  // one warp = one independent strip of 32*V columns, 2H of them halo
  constexpr int HS = P::HS;  // H rounded up to whole lanes
  a.strip = ((32 * V - 2 * HS) / VEC) * VEC;
  if (a.strip <= 0) return cudaErrorInvalidValue;
  a.xorg = floor_div(L.x0 - HS, VEC) * VEC;
  const int width = L.x1 - (a.xorg + HS);
  a.warps_x = std::max(1, (width + a.strip - 1) / a.strip);
  // strips whose 32V columns reach outside the interior (general path)
  {
    int nl = 0, nr = 0;
    for (int wx = 0; wx < a.warps_x && a.xorg + wx * a.strip < L.ix0; ++wx) ++nl;
    for (int wx = a.warps_x - 1; wx >= nl && a.xorg + wx * a.strip + 32 * V > L.ix1; --wx) ++nr;
    a.nl = nl;
    a.nr = nr;
    if (nl + nr >= a.warps_x) {  // every strip is slow: plain order
      a.nl = a.warps_x;
      a.nr = 0;
    }
    const int groups = (a.warps_x + NT / 32 - 1) / (NT / 32);
    a.gnl = (a.nl + NT / 32 - 1) / (NT / 32);
    a.gnr = std::max(0, groups - (a.warps_x - a.nr) / (NT / 32));  // incl. a partial last group
    if (a.gnl + a.gnr >= groups) a.gnl = groups, a.gnr = 0;
  }
  constexpr int NW = NT / 32;
  const int height = L.y1 - L.y0;
  // One wave of persistent CTAs; warps pull (strip, segment) items from a
  // counter. Segments: a few items per resident warp for load balance, each
  // at least 4x its warm-up (2 R*S rows + the S-iteration pipeline fill).
  auto kern = k1_stencil2d<T, R, S, KIND, V, NT, minb2d<T>(R, S)>;
  static int occ_by_dev[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  int occ = occ_by_dev[dev];
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0) != cudaSuccess || occ < 1) occ = 1;
    occ_by_dev[dev] = occ;
  }
  const int sms = device_sm_count();
  const int resident_warps = sms * occ * NW;
  // streaming shapes hand out CTA items (strip groups of NW strips), the
  // general path warp items (strips)
  constexpr bool kGroup = KIND != KGRAD && !(sizeof(T) == 8 && R >= 3) && P::GROUPED;
  constexpr bool kStreamPath = KIND != KGRAD && !(sizeof(T) == 8 && R >= 3);
  const int units = kGroup ? (a.warps_x + NW - 1) / NW : a.warps_x;
  const int edge_units = kGroup ? a.gnl + a.gnr : a.nl + a.nr;
  const int workers = kGroup ? sms * occ : resident_warps;
  // uniform segments: ipw items per worker, each >= 4x its warm-up
  const int min_seg_u = std::max(32, 4 * (2 * H + 2 * S * ((R + 1) / 2)));
  const int ipw = k1_items_per_warp_override() ? k1_items_per_warp_override() : 8;  // profiles/r02_guided/ipw_ab.txt
  const int ns_u = std::min(std::max(1, (ipw * workers + units - 1) / units), std::max(1, height / min_seg_u));
  const int seg_u = std::max(1, (height + ns_u - 1) / ns_u);
  if (k1_uniform_segments()) {
    a.seg_e = a.seg_b = a.seg_s = seg_u;
    a.nseg_e = a.nseg_b = (height + seg_u - 1) / seg_u;
    a.nseg_s = 0;
  } else {
    // guided: the same or shorter segments, the tail cut finer. Rows an item
    // recomputes besides its own: H warm-up rows, the pipeline fill
    // (2*ceil(R/2) rows per stage streaming, R+1 general) and ~6 rows' worth
    // of per-item setup latency
    const int ov = H + (kStreamPath ? 2 * S * ((R + 1) / 2) : S * (R + 1)) + 6;
    const K1SegPlan sp = k1_plan_segments(height, units, edge_units >= units ? units : edge_units, workers, ov,
                                          4.5, std::max(16, 2 * ov), seg_u);
    a.seg_e = sp.seg_e, a.nseg_e = sp.nseg_e;
    a.seg_b = sp.seg_b, a.nseg_b = sp.nseg_b;
    a.seg_s = sp.seg_s, a.nseg_s = sp.nseg_s;
  }
  a.counter = k1_next_counter(stream);
  if (!a.counter) return cudaErrorUnknown;
  const int ne = edge_units >= units ? units : edge_units;
  const int items = ne * a.nseg_e + (units - ne) * (a.nseg_b + a.nseg_s);
  const int ctas = std::max(1, std::min(sms * occ, kGroup ? items : (items + NW - 1) / NW));
  kern<<<ctas, NT, 0, stream>>>(a);
  return cudaGetLastError();
}

template <typename T, int R, int KIND, int S = 1>
cudaError_t launch_2d_s(const K1Launch& L, cudaStream_t stream) {
  if constexpr (S > maxs2d<T>(R)) {
    return cudaErrorInvalidValue;
  } else {
    if (L.steps == S) return launch_2d_fixed<T, R, S, KIND, v2d<T>(R)>(L, stream);
    return launch_2d_s<T, R, KIND, S + 1>(L, stream);
  }
}

template <typename T, int R>
cudaError_t launch_2d_r(const K1Launch& L, cudaStream_t stream) {
  if (L.steps < 1) return cudaErrorInvalidValue;
  switch (L.kind) {
    case KGRAD:
      if constexpr (R == 1) return launch_2d_s<T, 1, KGRAD>(L, stream);
      return cudaErrorInvalidValue;
    case KBOX: return launch_2d_s<T, R, KBOX>(L, stream);
    case KSTAR: return launch_2d_s<T, R, KSTAR>(L, stream);
  }
  return cudaErrorInvalidValue;
}

// per-(type, radius) entry points, each compiled in its own translation unit
cudaError_t launch_k1_2d_f32_r1(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r2(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r3(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r4(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r1(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r2(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r3(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r4(const K1Launch& L, cudaStream_t s);

}  // namespace so2dr_dev

// k1_2d_impl.cuh -- launch-side dispatch of the 2D K1 kernels (included by
// k1_2d_f32.cu / k1_2d_f64.cu so the two element types compile in parallel).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "k1_2d.cuh"
#include "k1_2d_p2.cuh"
#include "k1_launch.h"

namespace so2dr_dev {

constexpr int kThreads2D = 256;

// cells per thread (V) and the launch-bounds occupancy target per shape
template <typename T>
constexpr int v2d(int R) {
  return sizeof(T) == 4 ? 4 : (R <= 2 ? 2 : 4);
}
template <typename T>
constexpr int maxs2d(int R) {
  // (2R+1)^2 taps x S stages x 2R+1 unrolled phases grows fast: larger radii
  // fuse fewer steps per launch (the engine splits longer calls)
  return sizeof(T) == 4 ? (R == 1 ? 8 : R == 2 ? 4 : R == 3 ? 2 : 1) : (R == 1 ? 8 : R == 2 ? 4 : 1);
}

inline int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Tuning knob for experiments: SO2DR_K1_V=2 selects the 2-cell-per-thread
// variant of the fp32 radius-1 kernels (default 4).
inline int k1_v_override() {
  static int v = [] {
    const char* s = std::getenv("SO2DR_K1_V");
    return s ? std::atoi(s) : 0;
  }();
  return v;
}

// Experiment knob: SO2DR_K1_IMPL=p2 selects the paired-strip packed kernel
// (k1_2d_p2.cuh) for fp32 box/star, =pk the single-strip packed kernel.
inline int k1_impl_override() {
  static int v = [] {
    const char* s = std::getenv("SO2DR_K1_IMPL");
    if (!s) return 0;
    return std::strcmp(s, "p2") == 0 ? 2 : std::strcmp(s, "pk") == 0 ? 1 : std::strcmp(s, "hyb") == 0 ? 4 : 0;
  }();
  return v;
}

// Work items per resident warp (row segments x strips): more items balance
// the tail, longer segments amortise the R*S warm-up rows and the S-stage
// pipeline fill. Measured (profiles/r01_k1/ipw_*): launches over a whole grid
// (32768 rows) are best at 8 (6: -6%), the ~1500-row launches of the bench's
// d=64 chunks at 6 (8: -3%). SO2DR_K1_IPW=n overrides (experiments).
inline int k1_items_per_warp(int height) {
  static int v = [] {
    const char* s = std::getenv("SO2DR_K1_IPW");
    return s ? std::max(1, std::atoi(s)) : 0;
  }();
  if (v) return v;
  return height < 4096 ? 6 : 8;
}

template <typename T, int R, int S, int KIND, int V, int MINB,
          bool PACK = std::is_same_v<T, float> && KIND != KGRAD && V % 2 == 0, bool HYB = false>
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
  {
    const int64_t pb = L.pitch * static_cast<int64_t>(sizeof(T));
    a.cpb = pb % 16 == 0 ? 16 : pb % 8 == 0 ? 8 : 4;
  }
  // one warp = one independent strip of 32*V columns, 2H of them halo
  a.strip = ((32 * V - 2 * H) / VEC) * VEC;
  if (a.strip <= 0) return cudaErrorInvalidValue;
  a.xorg = floor_div(L.x0 - H, VEC) * VEC;
  const int width = L.x1 - (a.xorg + H);
  a.warps_x = std::max(1, (width + a.strip - 1) / a.strip);
  // strips whose 32V columns reach outside the interior (warp_ring in k1_item)
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
  }
  constexpr int NW = NT / 32;
  const int height = L.y1 - L.y0;
  // One wave of persistent CTAs; warps pull (strip, segment) items from a
  // counter. Segments: ~8 items per resident warp for load balance, but each
  // at least 6x its warm-up (R*S rows + S*(R+1) pipeline fill) long.
  constexpr bool packed = PACK;
  auto kern = [] {
    if constexpr (packed)
      return k1_stencil2d_pk<R, S, KIND, V, NT, MINB, HYB>;
    else
      return k1_stencil2d<T, R, S, KIND, V, NT, MINB, std::is_same_v<T, float> && KIND != KGRAD>;
  }();
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0) != cudaSuccess || occ < 1)
      occ = 1;
  }
  const int sms = device_sm_count();
  const int resident_warps = sms * occ * NW;
  const int min_seg = std::max(48, 6 * (H + S * (R + 1)));
  const int max_ns = std::max(1, height / min_seg);
  int ns = std::max(1, (k1_items_per_warp(height) * resident_warps + a.warps_x - 1) / a.warps_x);
  ns = std::min(ns, max_ns);
  a.seg = (height + ns - 1) / ns;
  a.nseg = (height + a.seg - 1) / a.seg;
  a.counter = k1_next_counter(stream);
  if (!a.counter) return cudaErrorUnknown;
  const int items = a.warps_x * a.nseg;
  const int ctas = std::max(1, std::min(sms * occ, (items + NW - 1) / NW));
  kern<<<ctas, NT, 0, stream>>>(a);
  return cudaGetLastError();
}

// Paired-strip launch (k1_2d_p2.cuh): one warp item = two strips x one row
// segment; same geometry rules as launch_2d_fixed.
template <int R, int S, int KIND, int V, int NT, int MINB>
cudaError_t launch_2d_p2(const K1Launch& L, cudaStream_t stream) {
  constexpr int H = R * S;
  constexpr int VEC = (V * 4) >= 16 ? 4 : V;
  using P = K1PlanP2<R, S, KIND, V, NT>;
  K1Args2D<float> a;
  a.in = static_cast<const float*>(L.in);
  a.out = static_cast<float*>(L.out);
  a.pitch = L.pitch;
  a.base = L.base;
  a.rows = L.rows;
  a.cols = L.cols;
  a.y0 = L.y0, a.y1 = L.y1, a.x0 = L.x0, a.x1 = L.x1;
  a.iy0 = L.iy0, a.iy1 = L.iy1, a.ix0 = L.ix0, a.ix1 = L.ix1;
  constexpr int E = 2 * R + 1;
  for (int i = 0; i < 81; ++i) a.w[i] = 0.f;
  if (L.w)
    for (int i = 0; i < E * E; ++i) a.w[i] = static_cast<float>(L.w[i]);
  {
    const int64_t pb = L.pitch * 4;
    a.cpb = pb % 16 == 0 ? 16 : pb % 8 == 0 ? 8 : 4;
  }
  a.strip = ((32 * V - 2 * H) / VEC) * VEC;
  if (a.strip <= 0) return cudaErrorInvalidValue;
  a.xorg = floor_div(L.x0 - H, VEC) * VEC;
  const int width = L.x1 - (a.xorg + H);
  a.warps_x = std::max(1, (width + a.strip - 1) / a.strip);
  {
    int nl = 0, nr = 0;
    for (int wx = 0; wx < a.warps_x && a.xorg + wx * a.strip < L.ix0; ++wx) ++nl;
    for (int wx = a.warps_x - 1; wx >= nl && a.xorg + wx * a.strip + 32 * V > L.ix1; --wx) ++nr;
    a.nl = nl;
    a.nr = nr;
  }
  constexpr int NW = NT / 32;
  const int height = L.y1 - L.y0;
  auto kern = k1_stencil2d_p2<R, S, KIND, V, NT, MINB>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    if (e != cudaSuccess) return e;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, P::SMEM) != cudaSuccess || occ < 1) occ = 1;
  }
  const int sms = device_sm_count();
  const int np = (a.warps_x + 1) / 2;
  const int resident_warps = sms * occ * NW;
  const int min_seg = std::max(48, 6 * (H + S * (R + 1)));
  const int max_ns = std::max(1, height / min_seg);
  int ns = std::max(1, (k1_items_per_warp(height) * resident_warps + np - 1) / np);
  ns = std::min(ns, max_ns);
  a.seg = (height + ns - 1) / ns;
  a.nseg = (height + a.seg - 1) / a.seg;
  a.counter = k1_next_counter(stream);
  if (!a.counter) return cudaErrorUnknown;
  const int items = np * a.nseg;
  const int ctas = std::max(1, std::min(sms * occ, (items + NW - 1) / NW));
  kern<<<ctas, NT, P::SMEM, stream>>>(a);
  return cudaGetLastError();
}

template <typename T, int R, int KIND, int S = 1>
cudaError_t launch_2d_s(const K1Launch& L, cudaStream_t stream) {
  if constexpr (S > maxs2d<T>(R)) {
    return cudaErrorInvalidValue;
  } else {
    if (L.steps == S) {
      if constexpr (sizeof(T) == 4 && R == 1 && KIND != KGRAD) {
        if (k1_v_override() == 2) return launch_2d_fixed<T, R, S, KIND, 2, 2>(L, stream);
        // 8 cells per lane (scalar FFMA; 198 registers at S = 4, 1 CTA/SM): 77% of
        // the steady-state loop's instructions are FFMA vs 68% at V = 4
        if constexpr (S <= 4) {
          if (k1_v_override() == 8 && k1_impl_override() != 1)
            return launch_2d_fixed<T, R, S, KIND, 8, 1, false>(L, stream);
        }
        // Paired-strip kernel (SO2DR_K1_IMPL=p2; S = 3..4 only: at S > 4 it needs
        // V = 2 and spills). In-core it is within noise of pk (+-3% at S = 4,
        // profiles/r01_k1); inside the bench pipeline (d=64, ~1500-row
        // launches) it was 20% slower per launch (0.54 vs 0.45 ms), so pk stays
        // the default. 128-thread CTAs, 3 per SM: <= 170 registers, no spill.
        if constexpr (S >= 3 && S <= 4) {
          if (k1_impl_override() == 2) return launch_2d_p2<R, S, KIND, 4, 128, 3>(L, stream);
        }

      }
      // fp32 box/star: the scalar-FFMA pipeline (k1_item) is the default. FFMA
      // reaches the same FMA rate as FFMA2 on this part (36.4 vs 36.9 TFMA/s,
      // profiles/r01_pcie/fma_peak.jsonl), and without register pairs ptxas
      // needs no IMAD.MOVs to assemble operands: +11-19% over the packed
      // kernel in-core (profiles/r01_k1/scalar_vs_pk.txt). SO2DR_K1_IMPL=pk
      // selects the packed FFMA2 kernel.
      // (the packed kernel is built for r <= 2 only: at r >= 3 its 2r+2-slot
      // ring outgrows the register file)
      if constexpr (sizeof(T) == 4 && KIND != KGRAD && R >= 3) {
        return launch_2d_fixed<T, R, S, KIND, v2d<T>(R), 1, false>(L, stream);
      } else {
        if constexpr (sizeof(T) == 4 && KIND != KGRAD) {
          // hybrid: FFMA2 where the operand pair is in registers, scalar FFMA
          // for the halo taps (SO2DR_K1_IMPL=hyb, experiment)
          if (k1_impl_override() == 4) return launch_2d_fixed<T, R, S, KIND, v2d<T>(R), 1, true, true>(L, stream);
          if (k1_impl_override() != 1) return launch_2d_fixed<T, R, S, KIND, v2d<T>(R), 1, false>(L, stream);
        }
        return launch_2d_fixed<T, R, S, KIND, v2d<T>(R), 1>(L, stream);
      }
    }
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

// k1_2d_stream.cuh -- K1 2D fast path: the streaming pipeline for work items
// that touch no pass-through cell (no ring column in the strip, no ring row in
// any stage's output range). Every iteration runs the same branch-free body,
// including the pipeline fill and drain; that is safe because a row a stage
// computes from rows outside its light cone (the fill's zero state, a stale
// ring slot, rows beyond the storage) never reaches a stored row: every output
// accumulator only ever receives taps from the rows of its own cone. The
// general path (k1_item in k1_2d.cuh) keeps the exact per-stage row ranges for
// the items that do touch the ring; it costs ~4.6x more instructions per
// iteration, which is why the fill and drain of short segments dominated the
// old kernel inside the bench pipeline (profiles/r02_k1).
//
// Same contract and per-point arithmetic as the reference's fused_kernel /
// stencil_row (proj/src/kernels.cpp:27-145, proj/src/stencil.cpp:120-144):
// every output point receives its taps in the canonical (dy, dx) order from a
// +0 start, so results are bit-identical.
//
// Row pairs. One iteration consumes two rows (P, P+1) in every stage, and a
// stage's accumulators are pairs Q[q] = (out q, out q+1), q = P (mod 2). An
// input value v at (row s, col x) contributes to out q with weight w(s-q, .)
// and to out q+1 with w(s-q-1, .): when both taps exist they are ONE packed
// FFMA2 with v as a broadcast scalar operand (SASS `FFMA2 Rd, Rv.F32,
// URw.F32x2, Rq`), the weight pair in uniform registers and the accumulator
// pair in place -- no operand moves. Box r=1: 24 FFMA2 + 24 FFMA per stage and
// iteration for 72 fmas (36% fewer FMA-pipe issue slots than scalar FFMA);
// each half of FFMA2 is an IEEE RN fma, bit-identical to __fmaf_rn. fp64 and
// r >= 3 (where the weight pairs outgrow the uniform registers) use the same
// pipeline with scalar fmas.
//
// Lag: stage u completes pair Q[P_u - 2C] (C = ceil(R/2)) after consuming
// (P_u, P_u+1); stage u+1 consumes that pair in the SAME iteration (stages
// run in ascending order), so P_{u+1} = P_u - 2C and the stored pair is
// Q[P0 - 2CS]. Accumulator slots rotate with period NSLOT = 2C+1 iterations
// (the loop is unrolled by NSLOT so every register index is static).
#pragma once

#include <type_traits>

#include "k1_2d.cuh"

namespace so2dr_dev {

template <typename T, int R, int KIND>
struct StreamPlan2D {
  static constexpr int C = (R + 1) / 2;      // per-stage lag in row pairs
  static constexpr int IMAX = (R + 1) / 2;   // farthest pair a new row starts
  static constexpr int NSLOT = C + IMAX + 1;  // live accumulator pairs per stage
  static constexpr bool PAIRED = std::is_same_v<T, float> && R <= 2;
  static constexpr bool tap(int dy, int dx) { return KIND == KBOX || dy == 0 || dx == 0; }
  static constexpr int first_dx(int dy) { return (KIND == KSTAR && dy != 0) ? 0 : -R; }
};

// ---- predicated memory helpers (no branches in the streaming loop) ----------
// cp.async of one lane's VB bytes (VB = V * sizeof(T), a multiple of 16 for
// every shape this path runs) into shared memory, with the largest pieces the
// global address allows (rows of an odd pitch start 8- or 4-byte aligned);
// nothing is copied when `ok` is false.
template <int VB>
__device__ __forceinline__ void cp_lane_pred(unsigned sdst, const void* g, bool ok) {
  static_assert(VB % 16 == 0, "whole 16-byte lane vectors");
  const unsigned al = static_cast<unsigned>(reinterpret_cast<uintptr_t>(g)) & 15u;
  const int p16 = ok && al == 0, p8 = ok && (al == 8), p4 = ok && (al & 7) != 0;
#pragma unroll
  for (int b = 0; b < VB; b += 16) {
    const char* gb = static_cast<const char*>(g) + b;
    asm volatile(
        "{\n .reg .pred q16, q8, q4;\n"
        " setp.ne.b32 q16, %2, 0;\n setp.ne.b32 q8, %3, 0;\n setp.ne.b32 q4, %4, 0;\n"
        " @q16 cp.async.cg.shared.global [%0], [%1], 16;\n"
        " @q8 cp.async.ca.shared.global [%0], [%1], 8;\n"
        " @q8 cp.async.ca.shared.global [%0+8], [%1+8], 8;\n"
        " @q4 cp.async.ca.shared.global [%0], [%1], 4;\n"
        " @q4 cp.async.ca.shared.global [%0+4], [%1+4], 4;\n"
        " @q4 cp.async.ca.shared.global [%0+8], [%1+8], 4;\n"
        " @q4 cp.async.ca.shared.global [%0+12], [%1+12], 4;\n}\n" ::"r"(sdst + b),
        "l"(gb), "r"(p16), "r"(p8), "r"(p4)
        : "memory");
  }
}

// Inner-item variants (8-byte aligned rows, lanes entirely valid or entirely
// outside the output columns): 8-byte pieces under one predicate.
template <int VB>
__device__ __forceinline__ void cp_lane8(unsigned sdst, const void* g, bool ok) {
#pragma unroll
  for (int b = 0; b < VB; b += 8)
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(sdst + b),
        "l"(static_cast<const char*>(g) + b), "r"((int)ok)
        : "memory");
}
template <typename T, int V>
__device__ __forceinline__ void store_lane8(T* dst, const T (&v)[V], bool ok) {
#pragma unroll
  for (int k = 0; k < V; k += 8 / (int)sizeof(T)) {
    if constexpr (sizeof(T) == 4)
      asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.global.v2.f32 [%0], {%1, %2};\n}\n" ::"l"(dst + k),
                   "f"(v[k]), "f"(v[k + 1]), "r"((int)ok)
                   : "memory");
    else
      asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(dst + k),
                   "d"(v[k]), "r"((int)ok)
                   : "memory");
  }
}

// Store the V cells of one lane (columns xt..xt+V-1 of the row at `dst`):
// vector stores when every cell is valid (16- or 8-byte, as the address
// allows), else per cell under `smask`; nothing when `ok` is false.
template <typename T, int V>
__device__ __forceinline__ void store_lane_pred(T* dst, const T (&v)[V], unsigned smask, bool ok) {
  constexpr unsigned full = (1u << V) - 1u;
  const unsigned al = static_cast<unsigned>(reinterpret_cast<uintptr_t>(dst)) & 15u;
  const bool whole = ok && smask == full;
  if constexpr (sizeof(T) == 4) {
    static_assert(V == 4, "fp32 lanes hold 4 cells");
    const int p16 = whole && al == 0, p8 = whole && al == 8;
    const unsigned pm = ok && !(whole && (al & 7) == 0) ? smask : 0u;
    asm volatile(
        "{\n .reg .pred q16, q8, c0, c1, c2, c3;\n .reg .b32 m;\n"
        " setp.ne.b32 q16, %5, 0;\n setp.ne.b32 q8, %6, 0;\n"
        " and.b32 m, %7, 1;\n setp.ne.b32 c0, m, 0;\n and.b32 m, %7, 2;\n setp.ne.b32 c1, m, 0;\n"
        " and.b32 m, %7, 4;\n setp.ne.b32 c2, m, 0;\n and.b32 m, %7, 8;\n setp.ne.b32 c3, m, 0;\n"
        " @q16 st.global.v4.f32 [%0], {%1, %2, %3, %4};\n"
        " @q8 st.global.v2.f32 [%0], {%1, %2};\n"
        " @q8 st.global.v2.f32 [%0+8], {%3, %4};\n"
        " @c0 st.global.f32 [%0], %1;\n @c1 st.global.f32 [%0+4], %2;\n"
        " @c2 st.global.f32 [%0+8], %3;\n @c3 st.global.f32 [%0+12], %4;\n}\n" ::"l"(dst),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "r"(p16), "r"(p8), "r"(pm)
        : "memory");
  } else {
    // fp64: every cell is 8-byte aligned; 16-byte pairs when the address allows
#pragma unroll
    for (int k = 0; k < V; k += 2) {
      const int p16 = whole && ((al + 8 * k) & 15) == 0;
      const unsigned pm = (ok && !p16) ? (smask >> k) & 3u : 0u;
      asm volatile(
          "{\n .reg .pred q16, c0, c1;\n .reg .b32 m;\n setp.ne.b32 q16, %3, 0;\n"
          " and.b32 m, %4, 1;\n setp.ne.b32 c0, m, 0;\n and.b32 m, %4, 2;\n setp.ne.b32 c1, m, 0;\n"
          " @q16 st.global.v2.f64 [%0], {%1, %2};\n"
          " @c0 st.global.f64 [%0], %1;\n @c1 st.global.f64 [%0+8], %2;\n}\n" ::"l"(dst + k),
          "d"(v[k]), "d"(v[k + 1]), "r"(p16), "r"(pm)
          : "memory");
    }
  }
}

// One work item (strip wx, row segment sg). EDGE = false: the strip owns no
// ring column and every row stages 1..S emit for the segment is interior (the
// caller checks). EDGE = true: pass-through cells exist -- after every stage
// the completed rows' ring cells (ring rows: all cells; ring columns: the
// lane's ring cells) are reset to the read buffer's value, which is the value
// of a pass-through cell at every step; loads are range-checked per element.
//
// Stage-0 rows. Inner items are processed by the whole CTA: its NW warps take
// NW adjacent strips of the same segment (a strip group), and the group's
// rows stream through a CTA ring filled by bulk copies (the TMA engine:
// cp.async.bulk + a `full` mbarrier per slot, tx-counted). One copy per row
// covers all NW strips (from the 16-byte-aligned address at or below the
// group's first column; rows that start 8 bytes off copy one extra chunk),
// so the lanes issue no per-lane copy instructions and the L2 sees
// whole-sector requests. The copy of iteration j is issued by warp j mod NW,
// PF iterations ahead, after every warp released the slot's previous use
// (an `empty` mbarrier with one arrival per warp). Each lane reads its V
// cells with two 8-byte LDS. EDGE items run per warp and keep per-lane
// range-checked cp.async (lanes may hang over the grid).
struct GroupRing {
  unsigned ring_s;   // shared address of the CTA ring (slot = 2 rows of rowb bytes)
  const char* ring;  // generic address of the same
  unsigned full_s;   // RING/2 `full` mbarriers (8 bytes apart)
  unsigned empty_s;  // RING/2 `empty` mbarriers
  unsigned rowb;     // bytes per ring row (16-byte multiple)
  int wcg;           // column of the group's first strip (lane 0 cell 0 of warp 0)
};

// Item modes: the stage-0 load path and the pass-through handling.
enum : int {
  kModeEdge = 0,   // per warp; pass-through cells; range-checked per-lane cp.async
  kModeLane = 1,   // per warp, inner; 8-byte per-lane cp.async (the FMA-bound depths)
  kModeGroup = 2,  // CTA strip group, inner; bulk-copy CTA ring (the HBM-bound depths)
};

template <typename T, int R, int S, int KIND, int V, int NT, int MODE>
__device__ __forceinline__ void k1_item_stream(const K1Args2D<T>& a, int wx, int OY0, int OY1, T* wring, const GroupRing& gr,
                                               unsigned& g_it) {
  using P = K1Plan2D<T, R, S, KIND, V, NT>;
  using SP = StreamPlan2D<T, R, KIND>;
  constexpr int E = 2 * R + 1, H = R * S;
  constexpr int C = SP::C, NS = SP::NSLOT;
  constexpr int RING_IT = P::RING / 2;  // ring depth in iterations (2 rows each)
  // prefetch distance: the lane ring refills the slot read one iteration
  // earlier; the CTA ring leaves one slot of slack between the slowest warp's
  // release and the refill
  constexpr bool EDGE = MODE == kModeEdge, GROUP = MODE == kModeGroup;
  constexpr int PF = GROUP ? RING_IT - 2 : RING_IT - 1;
  constexpr int NW = NT / 32;
  static_assert(P::RING % 2 == 0 && RING_IT >= 2, "ring holds whole row pairs");
  static_assert(KIND != KGRAD, "fast path: box / star");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const int wc0 = a.xorg + wx * a.strip;
  const int OX0 = max(wc0 + P::HS, a.x0);
  const int OX1 = min(wc0 + P::HS + a.strip, a.x1);
  const int sy0 = a.base, sy1 = a.base + a.rows;
  const int lo0 = max(OY0 - H, sy0), hi0 = min(OY1 + H, sy1);
  const int n_iter = (OY1 - lo0 + 2 * C * S + 1) / 2;
  const int xt = wc0 + lane * V;

  unsigned smask = 0, ringmask = 0, inmask = 0;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int x = xt + k;
    if (x >= OX0 && x < OX1) smask |= 1u << k;
    if (x >= 0 && x < a.cols) {
      inmask |= 1u << k;
      if (x < a.ix0 || x >= a.ix1) ringmask |= 1u << k;
    }
  }
  const bool warp_ring = EDGE && (wc0 < a.ix0 || wc0 + 32 * V > a.ix1);
  // pass-through: reset the ring cells of completed row y (inside storage)
  auto passthru = [&](int y, T(&v)[V]) SO2DR_INLINE {
    if (y < sy0 || y >= sy1) return;
    const bool ring_row = y < a.iy0 || y >= a.iy1;
    if (!ring_row && !warp_ring) return;
    const unsigned m = ring_row ? inmask : ringmask;
    const T* g = a.in + (int64_t)(y - sy0) * a.pitch + xt;
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (m & (1u << k)) v[k] = __ldg(g + k);
  };

  // ---- stage-0 rows ---------------------------------------------------------
  // (EDGE: per-lane cp.async ring in the warp's region, each lane reads back
  // only what it copied; inner: the CTA bulk-copy ring). ldp / bsrc = the
  // lane's / the group's first cell of the next row pair.
  T* my_ring = wring + lane * V;
  const unsigned ring_s = smem_u32(my_ring);
  constexpr unsigned ROWB = 32 * V * sizeof(T);  // one lane-ring row (32 lanes)
  const int64_t pitch2 = 2 * a.pitch;
  const T* ldp = a.in + xt + (int64_t)(lo0 - sy0) * a.pitch;
  // inner: byte offset of the group's first cell past the 16-byte boundary,
  // for the pair's first / second row (fixed per item: 2 rows = 16k bytes)
  const T* grp0 = a.in + gr.wcg + (int64_t)(lo0 - sy0) * a.pitch;
  const unsigned off0 = static_cast<unsigned>(reinterpret_cast<uintptr_t>(grp0)) & 15u;
  const unsigned off1 = static_cast<unsigned>(reinterpret_cast<uintptr_t>(grp0 + a.pitch)) & 15u;
  const unsigned gbytes = (NW * a.strip + 32 * V - a.strip) * sizeof(T);  // group row bytes
  const unsigned nb0 = (gbytes + off0 + 15u) & ~15u, nb1 = (gbytes + off1 + 15u) & ~15u;
  const T* bsrc = grp0;
  const unsigned g0 = g_it;
  // read cursors: slot address, its `full` barrier, phase parity
  unsigned rd_f = gr.full_s + 8u * (g0 % RING_IT);
  unsigned rd_s = gr.ring_s + (g0 % RING_IT) * 2u * gr.rowb;
  unsigned rd_par = (g0 / RING_IT) & 1u;
  const unsigned f_end = gr.full_s + 8u * RING_IT;
  const unsigned lane_off = (wc0 - gr.wcg) * sizeof(T) + lane * V * sizeof(T);
  if constexpr (GROUP) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  auto issue = [&](int it) SO2DR_INLINE {
    const int row = lo0 + 2 * it;
    if constexpr (GROUP) {
      if (it < n_iter && (it & (NW - 1)) == warp) {  // warp-uniform: the whole warp stays converged
        const unsigned gj = g0 + it, slot = gj % RING_IT;
        // the slot's previous use released by every warp (first use: parity 1 passes)
        mbar_wait_addr(gr.empty_s + 8u * slot, ((gj / RING_IT) & 1u) ^ 1u);
        const unsigned fb = gr.full_s + 8u * slot, dst = gr.ring_s + slot * 2u * gr.rowb;
        const unsigned n0 = row < hi0 ? nb0 : 0u, n1 = row + 1 < hi0 ? nb1 : 0u;
        // lane 0 arms the barrier and issues the row copies (predicated, no branch)
        asm volatile(
            "{\n .reg .pred p, p0, p1;\n setp.eq.u32 p, %7, 0;\n"
            " setp.ne.and.u32 p0, %3, 0, p;\n setp.ne.and.u32 p1, %5, 0, p;\n"
            " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%6], %8;\n"
            " @p0 cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%6];\n"
            " @p1 cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%4], %5, [%6];\n}\n" ::"r"(dst),
            "r"(dst + gr.rowb), "l"(reinterpret_cast<const char*>(bsrc) - off0), "r"(n0),
            "l"(reinterpret_cast<const char*>(bsrc + a.pitch) - off1), "r"(n1), "r"(fb), "r"(lane), "r"(n0 + n1)
            : "memory");
      }
      bsrc += pitch2;
    } else {
      const unsigned d = ring_s + ((2 * it) & (P::RING - 1)) * ROWB;
      if constexpr (MODE == kModeLane) {
        // inner strips need 8-byte aligned rows (checked by the caller): no
        // alignment test, 8-byte pieces
        cp_lane8<V * (int)sizeof(T)>(d, ldp, row < hi0);
        cp_lane8<V * (int)sizeof(T)>(d + ROWB, ldp + a.pitch, row + 1 < hi0);
      } else if (warp_ring) {  // lanes may hang over the padded grid
        T* dg = my_ring + ((2 * it) & (P::RING - 1)) * (32 * V);
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2)
          if (row + r2 < hi0) {
            const T* gr2 = ldp + (int64_t)r2 * a.pitch;
            const int cpb = row_cpb(gr2 - xt);
#pragma unroll
            for (int v = 0; v < V; v += P::VEC)
              issue_vec<T, P::VEC>(dg + r2 * 32 * V + v, gr2 + v, cpb, xt + v, a.pitch);
          }
      } else {
        cp_lane_pred<V * (int)sizeof(T)>(d, ldp, row < hi0);
        cp_lane_pred<V * (int)sizeof(T)>(d + ROWB, ldp + a.pitch, row + 1 < hi0);
      }
      cp_async_commit();
      ldp += pitch2;
    }
  };
#pragma unroll
  for (int i = 0; i < PF; ++i) issue(i);

  // stored pair: rows P0 - 2CS, P0 - 2CS + 1 (P0 = lo0 + 2 it)
  T* stp = a.out + xt + (int64_t)(lo0 - 2 * C * S - sy0) * a.pitch;

  // ---- carried state: S stages x NS accumulator pairs (lo row, hi row) ------
  T acc[S][NS][2][V];
#pragma unroll
  for (int u = 0; u < S; ++u)
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) acc[u][j][0][k] = acc[u][j][1][k] = T(0);

  auto body = [&](auto phase_tag, int it) SO2DR_INLINE {
    constexpr int PH = decltype(phase_tag)::value;
    issue(it + PF);
    T in0[2][V];
    if constexpr (GROUP) {
      mbar_wait_addr(rd_f, rd_par);
      const char* r0 = gr.ring + (rd_s - gr.ring_s) + off0 + lane_off;
      const char* r1 = r0 + gr.rowb + (off1 - off0);
      T x[2][V];
#pragma unroll
      for (int k = 0; k < V; k += 8 / (int)sizeof(T)) {  // 8-byte LDS (rows start 8-byte aligned)
        if constexpr (sizeof(T) == 4) {
          const float2 x0 = *reinterpret_cast<const float2*>(r0 + 4 * k);
          const float2 x1 = *reinterpret_cast<const float2*>(r1 + 4 * k);
          x[0][k] = x0.x, x[0][k + 1] = x0.y, x[1][k] = x1.x, x[1][k + 1] = x1.y;
        } else {
          x[0][k] = *reinterpret_cast<const T*>(r0 + 8 * k);
          x[1][k] = *reinterpret_cast<const T*>(r1 + 8 * k);
        }
      }
#pragma unroll
      for (int k = 0; k < V; ++k) in0[0][k] = x[0][k], in0[1][k] = x[1][k];
      // release the slot: every lane's LDS above is ordered before lane 0's
      // arrive (__syncwarp orders the warp's accesses; arrive is a release)
      __syncwarp();
      asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %1, 0;\n @p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n}\n" ::"r"(
                       gr.empty_s + (rd_f - gr.full_s)),
                   "r"(lane)
                   : "memory");
      rd_f += 8u;
      rd_s += 2u * gr.rowb;
      if (rd_f == f_end) rd_f = gr.full_s, rd_s = gr.ring_s, rd_par ^= 1u;
    } else {
      cp_async_wait<PF>();
      const T* src = my_ring + ((2 * it) & (P::RING - 1)) * (32 * V);
#pragma unroll
      for (int k = 0; k < V; ++k) in0[0][k] = src[k];
#pragma unroll
      for (int k = 0; k < V; ++k) in0[1][k] = src[32 * V + k];
    }
    constexpr int SC = (PH - C + NS) % NS;  // slot completed this iteration

#pragma unroll
    for (int u = 1; u <= S; ++u) {
      // input rows of stage u: the pair stage u-1 completed this iteration
      T sv[2][V + 2 * R];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int k = 0; k < V; ++k) sv[s][R + k] = (u == 1) ? in0[s][k] : acc[u - 2][SC][s][k];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          // lanes 0 / 31 receive their own values: the strip's outer halo
          sv[s][j] = __shfl_up_sync(0xffffffffu, sv[s][R + V - R + j], 1);
          sv[s][R + V + j] = __shfl_down_sync(0xffffffffu, sv[s][R + j], 1);
        }
      }
      T(&A)[NS][2][V] = acc[u - 1];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int i = -C; i <= SP::IMAX; ++i) {
          const int dlo = s - 2 * i, dhi = s - 2 * i - 1;
          const bool lo_in = dlo >= -R && dlo <= R, hi_in = dhi >= -R && dhi <= R;
          if (!lo_in && !hi_in) continue;
          const int sl = (PH + i + NS) % NS;
#pragma unroll
          for (int dx = -R; dx <= R; ++dx) {
            const bool tl = lo_in && SP::tap(dlo, dx), th = hi_in && SP::tap(dhi, dx);
            if (!tl && !th) continue;
            const bool lo_first = dlo == -R && dx == SP::first_dx(dlo);
            const bool hi_first = dhi == -R && dx == SP::first_dx(dhi);
            const T wl = tl ? a.w[(dlo + R) * E + dx + R] : T(0);
            const T wh = th ? a.w[(dhi + R) * E + dx + R] : T(0);
#pragma unroll
            for (int k = 0; k < V; ++k) {
              const T v = sv[s][R + k + dx];
              if constexpr (SP::PAIRED) {
                if (tl && th && !hi_first) {  // (hi's +0 start: two scalar fmas)
                  uint64_t q = pack2(A[sl][0][k], A[sl][1][k]);
                  uint64_t d;
                  asm("fma.rn.f32x2 %0, %1, %2, %3;"
                      : "=l"(d)
                      : "l"(pack2(v, v)), "l"(a.wp[(dlo + R - 1) * E + dx + R]), "l"(q));
                  unpack2(d, A[sl][0][k], A[sl][1][k]);
                  continue;
                }
              }
              if (tl) A[sl][0][k] = fma_rn(wl, v, lo_first ? T(0) : A[sl][0][k]);
              if (th) A[sl][1][k] = fma_rn(wh, v, hi_first ? T(0) : A[sl][1][k]);
            }
          }
        }
      }
      if constexpr (EDGE) {
        const int yu = lo0 + 2 * it - 2 * C * u;  // rows stage u completed
        passthru(yu, A[SC][0]);
        passthru(yu + 1, A[SC][1]);
      }
    }

    // stage S completed rows (P0 - 2CS, +1): store the ones inside [OY0, OY1)
    const int y = lo0 + 2 * it - 2 * C * S;
    if constexpr (!EDGE) {  // lanes all-valid or all-halo (caller checks)
      store_lane8<T, V>(stp, acc[S - 1][SC][0], smask && y >= OY0 && y < OY1);
      store_lane8<T, V>(stp + a.pitch, acc[S - 1][SC][1], smask && y + 1 >= OY0 && y + 1 < OY1);
    } else {
      store_lane_pred<T, V>(stp, acc[S - 1][SC][0], smask, y >= OY0 && y < OY1);
      store_lane_pred<T, V>(stp + a.pitch, acc[S - 1][SC][1], smask, y + 1 >= OY0 && y + 1 < OY1);
    }
    stp += pitch2;
  };

  int it = 0;
  while (it < n_iter) {
    [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
      ((it < n_iter ? (body(std::integral_constant<int, Ps>{}, it), ++it, void()) : void()), ...);
    }(std::make_integer_sequence<int, NS>{});
  }
  if constexpr (GROUP) g_it += n_iter;  // every issued slot was waited on
  else cp_async_wait<0>();
}

}  // namespace so2dr_dev

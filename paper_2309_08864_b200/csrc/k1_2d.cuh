// k1_2d.cuh -- K1: the k-step temporal-blocked 2D stencil kernel for sm_100a.
//
// Replaces the reference's fused_kernel (proj/src/kernels.cpp:27-145) and its
// per-row arithmetic stencil_row (proj/src/stencil.cpp:120-144).
//
// Contract (identical to one reference fused_kernel call): given the read
// buffer holding rows [base, base+rows) of the padded grid, write into the
// write buffer the state after S steps of every cell in `region`
// (rows [y0,y1) x cols [x0,x1)). Cells outside `interior` pass through.
// Per-point arithmetic is the reference's canonical chain (box: +0 then one
// FMA per tap in (dy, dx) ascending order; star: the same chain over on-axis
// taps; gradient: the pinned expression), so results are bit-identical.
//
// Design (AN5D-style streaming, B200-first):
//  * Every WARP is an independent pipeline: it owns a column strip of 32*V
//    cells (V consecutive cells per lane) and streams the input rows of its
//    row segment (plus R*S warm-up rows each side) from HBM exactly once.
//    x neighbours come from warp shuffles only; the strip's outer R*S columns
//    are the deliberately recomputed halo of temporal blocking (valid output
//    32V - 2RS columns). No shared-memory exchange and no __syncthreads in the
//    main loop, so the S stages of one iteration are independent instruction
//    streams the scheduler can overlap.
//  * The S time steps are S pipeline stages. Stage u consumes one row of stage
//    u-1 per iteration (emitted one iteration earlier) and keeps 2R+1 partial
//    accumulators (one per output row the consumed row contributes to). Rows
//    arrive in ascending order, so every output point receives its taps in
//    exactly the canonical (dy, dx) order: the partial accumulation is
//    bit-exact.
//  * Input rows are prefetched kRing-1 rows ahead with cp.async (LDGSTS, 16 B
//    when aligned) into a per-lane shared-memory ring that only the issuing
//    lane reads back (no barrier). Each input row is read from HBM once and
//    each output row written once per launch.
//  * The main loop is unrolled by 2R+1 so accumulator slot rotation is static
//    (no local-memory indexing), and the steady state (every stage consumes
//    and emits an interior row, no ring column in the strip) runs a variant
//    with all range checks compiled away.
//
// Three arithmetic variants share this pipeline (k1_2d_impl.cuh picks one):
//  * k1_stencil2d<..., SCALAR=true>: one scalar FFMA per tap -- the fp32 default
//    (FFMA reaches the FMA peak on sm_100 as well as FFMA2, and without register
//    pairs ptxas needs no operand moves: profiles/r01_k1/scalar_vs_pk.txt);
//  * k1_stencil2d_pk: packed FFMA2 on cell pairs (k, k+V/2) (SO2DR_K1_IMPL=pk);
//  * k1_stencil2d<double>: DFMA (fp64), and the gradient's pinned expression.
// The paired-strip FFMA2 kernel lives in k1_2d_p2.cuh (SO2DR_K1_IMPL=p2).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "k1_launch.h"
#include "k1_segplan.h"

namespace so2dr_dev {

template <typename T>
struct K1Args2D {
  const T* in;      // read buffer; storage row 0 == padded row `base`
  T* out;           // write buffer, same geometry
  int64_t pitch;    // elements per storage row (multiple of 32)
  int base, rows;   // storage rows [base, base+rows)
  int cols;         // padded width
  int y0, y1, x0, x1;
  int iy0, iy1, ix0, ix1;
  // Row segments (work items = unit x segment, DESIGN.md 4 "guided items"):
  // units that own ring columns take uniform segments of seg_e rows; inner
  // units take nseg_b big segments of seg_b rows from y0, then the rest of
  // the rows in small segments of seg_s (handed out last: they fill the
  // launch tail)
  int seg_e, nseg_e;
  int seg_b, nseg_b;
  int seg_s, nseg_s;
  int strip;        // output columns per warp
  int xorg;         // column of lane 0 cell 0 of warp 0 (aligned to VEC)
  int warps_x;      // strips along x
  int nl, nr;       // leading / trailing strips that own ring columns (slow path)
  int gnl, gnr;     // the same in strip groups (CTA items of the streaming path)
  int cpb;          // cp.async piece bytes (16/8/4): largest dividing the pitch
  int aligned8;     // both buffers 8-byte aligned and the pitch even (rows 8-byte aligned)
  unsigned* counter;  // work-item counter (zeroed before the launch)
  T w[81];          // (2R+1)^2 weights, canonical order
  // fp32 r <= 2: packed weight pairs {w(d, dx), w(d-1, dx)} for d = 1-R..R at
  // [(d+R-1)(2R+1) + dx+R], read by the fast path's FFMA2 from uniform registers
  uint64_t wp[20];
};

template <typename T>
__device__ __forceinline__ T fma_rn(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_rn<float>(float a, float b, float c) {
  return __fmaf_rn(a, b, c);
}
template <>
__device__ __forceinline__ double fma_rn<double>(double a, double b, double c) {
  return __fma_rn(a, b, c);
}
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// Packed fp32 pair helpers for FFMA2 (PTX fma.rn.f32x2, new in sm_100).
// The packing movs are register-pair renames the compiler folds into the
// FFMA2 operand swizzles (.F32x2.HI_LO / .LO_HI).
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
// {lo, hi} = {w * a0 + c.lo, w * a1 + c.hi}, each rounded once (RN)
__device__ __forceinline__ uint64_t fma2(float w, float a0, float a1, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pack2(w, w)), "l"(pack2(a0, a1)), "l"(c));
  return d;
}

// {lo, hi} = {w * a.lo + c.lo, w * a.hi + c.hi} on an already packed pair
__device__ __forceinline__ uint64_t fma2p(float w, uint64_t a, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pack2(w, w)), "l"(a), "l"(c));
  return d;
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- mbarrier + bulk copy (TMA engine) helpers -----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_addr(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, multiple of 16 bytes) that
// completes `bytes` on the mbarrier
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Copy the VEC consecutive elements at column x of one row, global -> shared,
// with cp.async pieces of `cpb` bytes (16, 8 or 4; the caller picks the
// largest the row's start address allows -- dense rows of odd-multiple
// pitches alternate 16- and 8-byte alignment). A piece that would cross the
// row end falls back to per-element copies of its in-row part; elements
// outside [0, pitch) are skipped.
template <typename T, int VEC>
__device__ __forceinline__ void issue_vec(T* dst, const T* src, int cpb, int x, int64_t pitch) {
  constexpr int VB = VEC * (int)sizeof(T);
  constexpr int EB = sizeof(T) >= 8 ? 8 : 4;  // one element
  auto piece = [&](auto bytes_tag) {
    constexpr int B = decltype(bytes_tag)::value;
    constexpr int PE = B / (int)sizeof(T) > 0 ? B / (int)sizeof(T) : 1;
#pragma unroll
    for (int b = 0, e = 0; b < VB; b += B, e += PE) {
      if (x + e >= 0 && x + e + PE <= pitch) {
        cp_async<B>(reinterpret_cast<char*>(dst) + b, reinterpret_cast<const char*>(src) + b);
      } else if constexpr (PE > 1) {
#pragma unroll
        for (int j = 0; j < PE; ++j)
          if (x + e + j >= 0 && x + e + j < pitch)
            cp_async<EB>(reinterpret_cast<char*>(dst) + b + j * EB,
                         reinterpret_cast<const char*>(src) + b + j * EB);
      }
    }
  };
  if (VB >= 16 && cpb >= 16)
    piece(std::integral_constant<int, 16>{});
  else if (VB >= 8 && cpb >= 8)
    piece(std::integral_constant<int, 8>{});
  else
    piece(std::integral_constant<int, EB>{});
}

// Largest cp.async piece (16/8/4 bytes) a row starting at `row_start` allows.
__device__ __forceinline__ int row_cpb(const void* row_start) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(row_start);
  return (a & 15) == 0 ? 16 : (a & 7) == 0 ? 8 : 4;
}

// Steady-state copy of a lane's VB bytes (VB = V * sizeof(T), all columns
// inside the row): the largest pieces (16/8/4 bytes) the lane's address
// allows (dense rows of an odd-multiple-of-8-byte pitch alternate 16/8). No
// per-element range checks.
template <int VB>
__device__ __forceinline__ void issue_inrow(void* dst, const void* src) {
  char* d = static_cast<char*>(dst);
  const char* g = static_cast<const char*>(src);
  if constexpr (VB >= 16) {
    if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
#pragma unroll
      for (int b = 0; b < VB; b += 16) cp_async<16>(d + b, g + b);
      return;
    }
  }
  if constexpr (VB >= 8) {
    if ((reinterpret_cast<uintptr_t>(g) & 7) == 0) {
#pragma unroll
      for (int b = 0; b < VB; b += 8) cp_async<8>(d + b, g + b);
      return;
    }
  }
#pragma unroll
  for (int b = 0; b < VB; b += 4) cp_async<4>(d + b, g + b);
}

template <typename T, int R, int S, int KIND, int V, int NT>
struct K1Plan2D {
  // prefetch ring depth (rows per lane; power of two; <= 32 KB of smem)
  static constexpr int RING = (V * (int)sizeof(T)) <= 16 ? 16 : 8;
  static constexpr int E = 2 * R + 1;
  static constexpr int H = R * S;
  // strip halo in columns: H rounded up to whole lanes, so every lane is
  // either entirely inside the strip's output columns or entirely halo
  static constexpr int HS = (H + V - 1) / V * V;
  static constexpr int NW = NT / 32;
  static constexpr int CPB = (V * (int)sizeof(T)) >= 16 ? 16 : V * (int)sizeof(T);  // copy bytes
  static constexpr int VEC = CPB / (int)sizeof(T);  // elements per copy / alignment unit
  static_assert(V % VEC == 0, "V must be a whole number of copy vectors");
  static_assert(R <= V, "warp-shuffle halo needs R <= V");
  // shared memory: NW per-warp cp.async rings (RING rows x 32 lanes x V),
  // aliased by the CTA bulk-copy ring of the streaming path (RING/2 slots x 2
  // rows x the strip group's columns + one 16-byte slack chunk); the CTA only
  // switches between the two at item boundaries (__syncthreads)
  static constexpr int LANE_RING_B = RING * 32 * V * (int)sizeof(T);
  static constexpr int GROUP_COLS = NW * (32 * V - 2 * HS) + 2 * HS;  // NW strips incl. halo
  static constexpr int CTA_ROWB = (GROUP_COLS * (int)sizeof(T) + 16 + 15) / 16 * 16;
  static constexpr int SMEM_B = ((NW * LANE_RING_B > RING * CTA_ROWB ? NW * LANE_RING_B : RING * CTA_ROWB) + 127) / 128 * 128;
  // HBM-bound depths (S <= 2) stream through the CTA bulk-copy ring in strip
  // groups; the FMA-bound depths keep per-warp items (lockstep warps of a
  // group contend for the FMA pipe: 1701 vs 2184 GCell/s at box2d1r k=4,
  // profiles/r02_k1)
  static constexpr bool GROUPED = S <= 2;
  static constexpr int NACC = (KIND == KGRAD) ? 0 : S;
  static constexpr int NGR = (KIND == KGRAD) ? S : 0;
};

// One work item = (strip wx, row segment sg) processed by one warp; `wring`
// is the warp's shared ring (each lane uses its own slots only).
template <typename T, int R, int S, int KIND, int V, int NT, bool SCALAR = false>
__device__ __forceinline__ void k1_item(const K1Args2D<T>& a, int wx, int OY0, int OY1, T* wring) {
  using P = K1Plan2D<T, R, S, KIND, V, NT>;
  constexpr int E = P::E, H = P::H, VEC = P::VEC;
  constexpr int kRing = P::RING;
  const int tid = threadIdx.x, lane = tid & 31;
  constexpr bool live = true;

  // ---- warp geometry ------------------------------------------------------
  const int wc0 = a.xorg + wx * a.strip;  // column of lane 0 cell 0
  const int OX0 = max(wc0 + P::HS, a.x0);
  const int OX1 = min(wc0 + P::HS + a.strip, a.x1);
  const int sy0 = a.base, sy1 = a.base + a.rows;
  const int lo0 = max(OY0 - H, sy0), hi0 = min(OY1 + H, sy1);
  const int n_iter = OY1 - lo0 + S * (R + 1);
  const int xt = wc0 + lane * V;  // this lane's first column

  // rows produced by each stage: [lo_u, hi_u)
  int lo[S + 1], hi[S + 1];
#pragma unroll
  for (int u = 0; u <= S; ++u) {
    lo[u] = max(OY0 - R * (S - u), sy0);
    hi[u] = min(OY1 + R * (S - u), sy1);
  }

  // per-lane column masks: pass-through (ring / outside the grid) and store
  unsigned ringmask = 0, smask = 0;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int x = xt + k;
    if (x < a.ix0 || x >= a.ix1) ringmask |= 1u << k;
    if (live && x >= OX0 && x < OX1) smask |= 1u << k;
  }
  // whole copy vectors inside [0, pitch) are loaded (a lane may straddle
  // column 0 when V > VEC, e.g. fp64 with V=4)
  unsigned lmask = 0;
#pragma unroll
  for (int v = 0; v < V; v += VEC)
    if (xt + v >= 0 && xt + v < a.pitch) lmask |= 1u << v;
  // warp-uniform: does any lane own a pass-through column?
  const bool warp_ring = wc0 < a.ix0 || wc0 + 32 * V > a.ix1;

  // carried state
  T cur[S][V];                                // stage 0..S-1 emitted row (own cells)
  T acc[P::NACC > 0 ? P::NACC : 1][E][V];     // box/star partial accumulators
  T grow[P::NGR > 0 ? P::NGR : 1][3][V + 2];  // gradient row window (with x halo)
#pragma unroll
  for (int u = 0; u < S; ++u)
#pragma unroll
    for (int k = 0; k < V; ++k) cur[u][k] = T(0);

  // ---- prefetch (each lane reads back only what it copied: no barrier) ------
  T* my_ring = wring + lane * V;
  const T* src_col = a.in + xt;
  auto issue = [&](int row) SO2DR_INLINE {
    const bool ok = row < hi0;  // rows below lo0 never requested
    T* dst = my_ring + (row & (kRing - 1)) * (32 * V);
    const T* src = src_col + (int64_t)(row - sy0) * a.pitch;
    const int cpb = row_cpb(a.in + (int64_t)(row - sy0) * a.pitch);  // warp-uniform
#pragma unroll
    for (int v = 0; v < V; v += VEC)
      if (ok) issue_vec<T, VEC>(dst + v, src + v, cpb, xt + v, a.pitch);
    cp_async_commit();
  };
  // steady-state addressing off a running row offset (no 64-bit multiplies
  // per row): off = (row0 - sy0) * pitch, advanced by one row per iteration;
  // load row = row0 + kRing - 1, store row = row0 - S(R+1)
  int64_t off = (int64_t)(lo0 - sy0) * a.pitch;
  const T* ld_lane = src_col + (int64_t)(kRing - 1) * a.pitch;
  T* st_lane = a.out + xt - (int64_t)(S * (R + 1)) * a.pitch;
  auto issue_fast = [&](int row) SO2DR_INLINE {
    if (row < hi0) issue_inrow<V * (int)sizeof(T)>(my_ring + (row & (kRing - 1)) * (32 * V), ld_lane + off);
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < kRing - 1; ++d) issue(lo0 + d);

  const T* __restrict__ gin = a.in;
  T* __restrict__ gout = a.out;

  // pass-through value of cell (row, xt+k) from the read buffer
  auto passthru = [&](int row, int k) SO2DR_INLINE -> T {
    const int x = xt + k;
    if (x < 0 || x >= a.cols) return T(0);
    return __ldg(gin + (int64_t)(row - sy0) * a.pitch + x);
  };

  // One pipeline iteration at compile-time phase PH = it mod E. FAST = steady
  // state: every stage consumes and emits an interior row and the strip owns
  // no pass-through column, so all range checks compile away.
  auto body = [&](auto phase_tag, auto fast_tag, int it) SO2DR_INLINE {
    constexpr int PH = decltype(phase_tag)::value;
    constexpr bool FAST = decltype(fast_tag)::value;
    const int row0 = lo0 + it;

    // stages in descending order: stage u consumes cur[u-1] (emitted by stage
    // u-1 in the previous iteration) before stage u-1 overwrites it.
#pragma unroll
    for (int u = S; u >= 1; --u) {
      const int A = row0 - u - (u - 1) * R;  // row consumed by stage u
      const int Erow = A - R;                // row emitted by stage u
      const bool consume = FAST || (A >= lo[u - 1] && A < hi[u - 1]);
      const bool emit = FAST || (Erow >= lo[u] && Erow < hi[u]);

      // (shuffles run unconditionally: warp-convergent by construction)
      T seg[V + 2 * R];
#pragma unroll
      for (int k = 0; k < V; ++k) seg[R + k] = cur[u - 1][k];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        // lanes 0 / 31 receive their own values: the strip's outer halo,
        // finite garbage that never reaches a valid output column
        seg[j] = __shfl_up_sync(0xffffffffu, cur[u - 1][V - R + j], 1);
        seg[R + V + j] = __shfl_down_sync(0xffffffffu, cur[u - 1][j], 1);
      }

      T outv[V];
      if constexpr (KIND == KGRAD) {
        // rows: slot PH = A (just consumed), PH-1 = A-1 (centre), PH-2 = A-2 (north)
        constexpr int sA = PH % 3, sC = (PH + 2) % 3, sN = (PH + 1) % 3;
        if (consume) {
#pragma unroll
          for (int k = 0; k < V + 2; ++k) grow[u - 1][sA][k] = seg[k];
        }
        if (emit) {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const T c = grow[u - 1][sC][k + 1];
            const T dn = sub_rn(grow[u - 1][sN][k + 1], c);
            const T ds = sub_rn(grow[u - 1][sA][k + 1], c);
            const T de = sub_rn(grow[u - 1][sC][k + 2], c);
            const T dw = sub_rn(grow[u - 1][sC][k], c);
            const T sum = add_rn(add_rn(add_rn(dn, ds), de), dw);
            outv[k] = add_rn(c, mul_rn(T(0.25), sum));
          }
        }
      } else {
        if (consume) {
#pragma unroll
          for (int m = 0; m < E; ++m) {
            const int dy = m - R;                 // A contributes at dy to row A-dy
            const int sl = (PH - m + 2 * E) % E;  // slot of output row A+R-m
            if constexpr (sizeof(T) == 4 && V % 2 == 0 && !SCALAR) {
              // fp32: two cells per FFMA2 (fma.rn.f32x2, sm_100a); each half is
              // an IEEE fma with round-to-nearest, so the chain is bit-identical
              // to the scalar __fmaf_rn chain. Cells are paired (k, k+V/2), not
              // (k, k+1): then the operand pair for every dx, (s[k+dx],
              // s[k+V/2+dx]), is the same register pair the previous stage
              // emitted, except the 2R pairs that take a shuffled halo value --
              // so almost no register moves are needed to form operands.
              constexpr int HV = V / 2;
#pragma unroll
              for (int k = 0; k < HV; ++k) {
                uint64_t x = (m == 0) ? 0ull : pack2(acc[u - 1][sl][k], acc[u - 1][sl][k + HV]);
                if constexpr (KIND == KBOX) {
#pragma unroll
                  for (int dx = -R; dx <= R; ++dx)
                    x = fma2(a.w[(dy + R) * E + dx + R], seg[R + k + dx], seg[R + k + HV + dx], x);
                } else if (dy != 0) {
                  x = fma2(a.w[(dy + R) * E + R], seg[R + k], seg[R + k + HV], x);
                } else {
#pragma unroll
                  for (int dx = -R; dx <= R; ++dx)
                    x = fma2(a.w[R * E + dx + R], seg[R + k + dx], seg[R + k + HV + dx], x);
                }
                unpack2(x, acc[u - 1][sl][k], acc[u - 1][sl][k + HV]);
              }
            } else {
#pragma unroll
            for (int k = 0; k < V; ++k) {
              T x = (m == 0) ? T(0) : acc[u - 1][sl][k];
              if constexpr (KIND == KBOX) {
#pragma unroll
                for (int dx = -R; dx <= R; ++dx)
                  x = fma_rn(a.w[(dy + R) * E + dx + R], seg[R + k + dx], x);
              } else {  // star: on-axis taps only
                if (dy != 0) {
                  x = fma_rn(a.w[(dy + R) * E + R], seg[R + k], x);
                } else {
#pragma unroll
                  for (int dx = -R; dx <= R; ++dx)
                    x = fma_rn(a.w[R * E + dx + R], seg[R + k + dx], x);
                }
              }
              acc[u - 1][sl][k] = x;
            }
            }
          }
        }
        if (emit) {
          constexpr int se = (PH - 2 * R + 2 * E) % E;  // slot of row A-R
#pragma unroll
          for (int k = 0; k < V; ++k) outv[k] = acc[u - 1][se][k];
        }
      }

      if (emit) {
        if constexpr (!FAST) {
          if (Erow < a.iy0 || Erow >= a.iy1) {
#pragma unroll
            for (int k = 0; k < V; ++k) outv[k] = passthru(Erow, k);
          } else if (ringmask) {
#pragma unroll
            for (int k = 0; k < V; ++k)
              if (ringmask & (1u << k)) outv[k] = passthru(Erow, k);
          }
        }
        if (u == S) {
          T* dst = FAST ? st_lane + off : gout + (int64_t)(Erow - sy0) * a.pitch + xt;
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (smask & (1u << k)) dst[k] = outv[k];
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) cur[u][k] = outv[k];
        }
      }
    }

    // stage 0: row lo0 + it arrives from the cp.async ring
    if constexpr (FAST)
      issue_fast(row0 + kRing - 1);
    else
      issue(row0 + kRing - 1);
    cp_async_wait<kRing - 1>();
    if (FAST || row0 < hi0) {
      const T* src = my_ring + (row0 & (kRing - 1)) * (32 * V);
#pragma unroll
      for (int k = 0; k < V; ++k) cur[0][k] = src[k];
    }
    off += a.pitch;
  };

  // ---- steady-state window [f_lo, f_hi): every stage consumes a stored row
  // and emits an interior row, stage 0 still has rows to load.
  int f_lo = 0, f_hi = hi0 - lo0;
#pragma unroll
  for (int u = 1; u <= S; ++u) {
    const int c = lo0 - u - (u - 1) * R;  // A_u(it) = it + c
    f_lo = max(f_lo, lo[u - 1] - c);
    f_hi = min(f_hi, hi[u - 1] - c);
    f_lo = max(f_lo, max(lo[u], a.iy0) + R - c);
    f_hi = min(f_hi, min(hi[u], a.iy1) + R - c);
  }
  if (warp_ring) f_hi = f_lo;

  int it = 0;
  auto run_general = [&](int stop) SO2DR_INLINE {
    while (it < stop) {
      [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
        ((it < stop ? (body(std::integral_constant<int, Ps>{}, std::false_type{}, it), ++it, void())
                    : void()),
         ...);
      }(std::make_integer_sequence<int, E>{});
    }
  };
  const int fl = (f_lo + E - 1) / E * E;  // phase-aligned start of the fast loop
  if (f_hi - fl >= E) {
    run_general(fl);
    while (it + E <= f_hi) {
      [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
        ((body(std::integral_constant<int, Ps>{}, std::true_type{}, it), ++it), ...);
      }(std::make_integer_sequence<int, E>{});
    }
  }
  run_general(n_iter);
  cp_async_wait<0>();
}


// Work item -> (strip, output rows [oy0, oy1)). The strips that own ring
// columns run the range-checked edge pipeline and cost several times a
// steady-state item, so they are handed out FIRST (longest items first):
// fetched last they left one SM running alone for ~25% of the launch
// (profiles/r01_baseline/k1_full.json: SM active avg 73.5% of elapsed). The
// inner units' big segments come next and their small segments last, so the
// launch ends on short items (k1_plan_segments).
template <typename T>
__device__ __forceinline__ int k1_items_total(const K1Args2D<T>& a, int units) {
  const int nl = units == a.warps_x ? a.nl : a.gnl, nr = units == a.warps_x ? a.nr : a.gnr;
  return k1_seg_items(K1SegPlan{a.seg_e, a.nseg_e, a.seg_b, a.nseg_b, a.seg_s, a.nseg_s}, units, nl + nr);
}

template <typename T>
__device__ __forceinline__ void k1_item_coords(const K1Args2D<T>& a, int item, int& wx, int& oy0, int& oy1,
                                               int units) {
  // units: strips (per-warp items) or strip groups (CTA items); the leading /
  // trailing units that own ring columns come first
  const int nl = units == a.warps_x ? a.nl : a.gnl, nr = units == a.warps_x ? a.nr : a.gnr;
  k1_seg_decode(K1SegPlan{a.seg_e, a.nseg_e, a.seg_b, a.nseg_b, a.seg_s, a.nseg_s}, item, units, nl, nr, a.y0, a.y1,
                wx, oy0, oy1);
}

}  // namespace so2dr_dev

#include "k1_2d_stream.cuh"

namespace so2dr_dev {

// Persistent warps with dynamic work distribution: every warp of a one-wave
// grid fetches (strip, segment) items from an atomic counter, so the SMs stay
// busy until the last item (no partial last wave). Items that touch no
// pass-through cell run the branch-free streaming path (k1_2d_stream.cuh);
// the others the range-checked general path (k1_item). The last warp to
// leave re-arms the counter pair for the next launch that uses it, so no
// memset is enqueued per launch.
template <typename T, int R, int S, int KIND, int V, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k1_stencil2d(const K1Args2D<T> a) {
  using P = K1Plan2D<T, R, S, KIND, V, NT>;
  constexpr int NW = NT / 32;
  constexpr int H = R * S;
  __shared__ __align__(128) unsigned char smem[P::SMEM_B];
  __shared__ __align__(8) uint64_t bars[2][P::RING / 2];
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* wring = reinterpret_cast<T*>(smem + warp * P::LANE_RING_B);
  // streaming shapes (fp32 / fp64 r <= 2): the fp64 r >= 3 streaming state
  // outgrows the register file, so those (and the gradient) stay per warp
  constexpr bool kStream = KIND != KGRAD && !(sizeof(T) == 8 && R >= 3);
  if constexpr (kStream && P::GROUPED) {
    // CTA work items = (strip group of NW strips, row segment)
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < P::RING / 2; ++i) {
        mbar_init(&bars[0][i], 1);   // full: the issuing lane's expect_tx
        mbar_init(&bars[1][i], NW);  // empty: one release per warp
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    GroupRing gr;
    gr.ring_s = smem_u32(smem);
    gr.ring = reinterpret_cast<const char*>(smem);
    gr.full_s = smem_u32(&bars[0][0]);
    gr.empty_s = smem_u32(&bars[1][0]);
    gr.rowb = P::CTA_ROWB;
    unsigned g_it = 0;  // CTA-ring slots consumed (identical in every warp)
    const int groups = (a.warps_x + NW - 1) / NW;
    const int total = k1_items_total(a, groups);
    for (;;) {
      __syncthreads();  // every warp done with the previous item (and s_item)
      if (threadIdx.x == 0) s_item = static_cast<int>(atomicAdd(a.counter, 1u));
      __syncthreads();
      const int item = s_item;
      if (item >= total) break;
      int gx, OY0, OY1;
      k1_item_coords(a, item, gx, OY0, OY1, groups);
      const int wx0 = gx * NW;
      const int wc0 = a.xorg + wx0 * a.strip;
      // inner group: NW whole strips, no pass-through cell, rows stage 1 emits
      // (the widest stage range) all interior, 8-byte aligned rows, output
      // columns on lane boundaries, and the bulk copy's 16-byte slack inside
      // the row
      const int lo1 = max(OY0 - (H - R), a.base), hi1 = min(OY1 + (H - R), a.base + a.rows);
      const int wce = wc0 + (NW - 1) * a.strip + 32 * V;  // group's end column
      const int OX0 = max(wc0 + P::HS, a.x0), OX1 = min(wce - P::HS, a.x1);
      const bool lanes_whole = OX0 >= OX1 || ((OX0 - wc0) % V == 0 && (OX1 - wc0) % V == 0);
      const bool inner = wx0 + NW <= a.warps_x && wc0 >= a.ix0 && wce <= a.ix1 && lo1 >= a.iy0 &&
                         hi1 <= a.iy1 && wce * (int)sizeof(T) + 16 <= a.cols * (int)sizeof(T) && a.aligned8 &&
                         lanes_whole;
      if (inner) {
        gr.wcg = wc0;
        k1_item_stream<T, R, S, KIND, V, NT, kModeGroup>(a, wx0 + warp, OY0, OY1, wring, gr, g_it);
      } else if (wx0 + warp < a.warps_x) {
        k1_item_stream<T, R, S, KIND, V, NT, kModeEdge>(a, wx0 + warp, OY0, OY1, wring, gr, g_it);
      }
    }
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.counter + 1, 1u) == gridDim.x - 1) {
        a.counter[0] = 0u;
        a.counter[1] = 0u;
        __threadfence();
      }
    }
  } else if constexpr (kStream) {
    // per-warp work items = (strip, row segment) on the streaming path
    GroupRing gr{};
    unsigned g_it = 0;
    const int total = k1_items_total(a, a.warps_x);
    for (;;) {
      int item = 0;
      if (lane == 0) item = static_cast<int>(atomicAdd(a.counter, 1u));
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= total) break;
      int wx, OY0, OY1;
      k1_item_coords(a, item, wx, OY0, OY1, a.warps_x);
      const int wc0 = a.xorg + wx * a.strip;
      const int lo1 = max(OY0 - (H - R), a.base), hi1 = min(OY1 + (H - R), a.base + a.rows);
      const int OX0 = max(wc0 + P::HS, a.x0), OX1 = min(wc0 + P::HS + a.strip, a.x1);
      const bool lanes_whole = OX0 >= OX1 || ((OX0 - wc0) % V == 0 && (OX1 - wc0) % V == 0);
      const bool inner = wc0 >= a.ix0 && wc0 + 32 * V <= a.ix1 && lo1 >= a.iy0 && hi1 <= a.iy1 && a.aligned8 &&
                         lanes_whole;
      if (inner)
        k1_item_stream<T, R, S, KIND, V, NT, kModeLane>(a, wx, OY0, OY1, wring, gr, g_it);
      else
        k1_item_stream<T, R, S, KIND, V, NT, kModeEdge>(a, wx, OY0, OY1, wring, gr, g_it);
    }
    if (lane == 0) {
      __threadfence();
      const unsigned nw = gridDim.x * NW;
      if (atomicAdd(a.counter + 1, 1u) == nw - 1) {
        a.counter[0] = 0u;
        a.counter[1] = 0u;
        __threadfence();
      }
    }
  } else {
    // per-warp work items = (strip, row segment): general path
    const int total = k1_items_total(a, a.warps_x);
    for (;;) {
      int item = 0;
      if (lane == 0) item = static_cast<int>(atomicAdd(a.counter, 1u));
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= total) break;
      int wx, OY0, OY1;
      k1_item_coords(a, item, wx, OY0, OY1, a.warps_x);
      k1_item<T, R, S, KIND, V, NT, true>(a, wx, OY0, OY1, wring);
    }
    // The last warp to leave re-arms the counter pair for the next launch
    // that uses it (no memset per launch).
    if (lane == 0) {
      __threadfence();
      const unsigned nw = gridDim.x * NW;
      if (atomicAdd(a.counter + 1, 1u) == nw - 1) {
        a.counter[0] = 0u;
        a.counter[1] = 0u;
        __threadfence();
      }
    }
  }
}

}  // namespace so2dr_dev

// k1_2d_p2.cuh -- K1 (2D, fp32, box/star), PAIRED-STRIP variant for sm_100a.
//
// Same contract and per-point arithmetic as k1_item_pk (k1_2d.cuh): one
// reference fused_kernel call (proj/src/kernels.cpp:27-145), canonical
// (dy, dx) FMA chains of stencil_row (proj/src/stencil.cpp:120-144),
// bit-identical results.
//
// Why a second packed variant: in k1_item_pk a lane packs its OWN cells
// (k, k+V/2) into FFMA2 operand pairs, so the two x-halo pairs of every
// consumed row, (halo_left, cell V/2-1) and (cell V/2, halo_right), have to
// be assembled with register moves -- and ptxas spends ~90 IMAD.MOV/MOV per
// 144 FFMA2 on them and on re-forming pairs under register pressure
// (profiles/r01_baseline, tools/sass_loops.py). IMAD.MOV issues on the same
// FMA pipe as FFMA2.
//
// Here every warp runs TWO column strips in lockstep, A (strip q) and B
// (strip W-1-q), over the same rows: pair k of a lane is (A cell k, B cell k).
// The operand pair of tap dx is then always (A cell k+dx, B cell k+dx): an
// existing pair for in-lane neighbours, and for the halo the two shuffle
// results, which ptxas writes straight into an aligned register pair. No
// moves are needed to form operands. Both strips share every row-dependent
// decision (stage ranges, steady-state window), so the paired pipeline is the
// single-strip pipeline with 2x the work per instruction; column-dependent
// masks (ring pass-through, store window) are kept per strip. Pairing q with
// W-1-q puts the two ring-column strips of a row band into the same item.
#pragma once

#include "k1_2d.cuh"

namespace so2dr_dev {

template <int R, int S, int KIND, int V, int NT>
struct K1PlanP2 {
  static constexpr int RING = 8;  // prefetch ring depth (rows)
  // dynamic shared memory: ring[RING][2][NT * V] floats
  static constexpr size_t SMEM = sizeof(float) * RING * 2 * NT * V;
  static constexpr int E = 2 * R + 1;
  static constexpr int H = R * S;
  static_assert(R <= V, "warp-shuffle halo needs R <= V");
  static_assert(KIND != KGRAD, "paired packed path: box/star");
};

__device__ __forceinline__ float lo_of(uint64_t p) {
  float lo, hi;
  unpack2(p, lo, hi);
  return lo;
}
__device__ __forceinline__ float hi_of(uint64_t p) {
  float lo, hi;
  unpack2(p, lo, hi);
  return hi;
}

template <int R, int S, int KIND, int V, int NT>
__device__ __forceinline__ void k1_item_p2(const K1Args2D<float>& a, int q, int sg, float* ring) {
  using T = float;
  using P = K1PlanP2<R, S, KIND, V, NT>;
  constexpr int E = P::E, H = P::H, kRing = P::RING;
  constexpr int VEC = (V * 4) % 16 == 0 ? 4 : (V * 4) % 8 == 0 ? 2 : 1;  // cp.async unit (elements)
  const int tid = threadIdx.x, lane = tid & 31;

  // ---- geometry: rows shared, columns per strip ------------------------------
  const int wxa = q, wxb = a.warps_x - 1 - q;
  const int wc0[2] = {a.xorg + wxa * a.strip, a.xorg + wxb * a.strip};
  const int OY0 = a.y0 + sg * a.seg;
  const int OY1 = min(OY0 + a.seg, a.y1);
  const int sy0 = a.base, sy1 = a.base + a.rows;
  const int lo0 = max(OY0 - H, sy0), hi0 = min(OY1 + H, sy1);
  const int n_iter = OY1 - lo0 + S * (R + 1);
  int xt[2];
  unsigned ringmask[2] = {0u, 0u}, smask[2] = {0u, 0u};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    xt[h] = wc0[h] + lane * V;
    const int OX0 = max(wc0[h] + H, a.x0);
    const int OX1 = min(wc0[h] + H + a.strip, a.x1);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int x = xt[h] + k;
      if (x < a.ix0 || x >= a.ix1) ringmask[h] |= 1u << k;
      if (x >= OX0 && x < OX1) smask[h] |= 1u << k;
    }
  }
  if (wxb == wxa) smask[1] = 0u;  // odd strip count: the middle strip runs twice, stored once
  const bool warp_ring = wc0[0] < a.ix0 || wc0[0] + 32 * V > a.ix1 || wc0[1] < a.ix0 ||
                         wc0[1] + 32 * V > a.ix1;

  int lo[S + 1], hi[S + 1];
#pragma unroll
  for (int u = 0; u <= S; ++u) {
    lo[u] = max(OY0 - R * (S - u), sy0);
    hi[u] = min(OY1 + R * (S - u), sy1);
  }

  float c0a[V], c0b[V];  // stage-0 (loaded) row: A cells, B cells
  uint64_t ap[S][E][V];  // partial accumulators; stage u's emitted row stays in its slot
#pragma unroll
  for (int k = 0; k < V; ++k) c0a[k] = c0b[k] = 0.f;
#pragma unroll
  for (int u = 0; u < S; ++u)
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int k = 0; k < V; ++k) ap[u][e][k] = 0ull;

  // ---- prefetch: each lane reads back only what it copied (no barrier) -------
  // Ring slot per lane: A's V cells then B's V cells, each copied with the
  // widest cp.async the row alignment allows (an interleaved (A_k, B_k) layout
  // needs 4-byte copies: 4x the L1 wavefronts, MIO-throttled, profiles/r01_k1).
  // Stage 1 therefore consumes the loaded row as two scalar vectors (FFMA into
  // the halves of its pair accumulators); stages 2..S run on pairs (FFMA2).
  auto slot = [&](int row, int h) -> T* { return ring + ((row & (kRing - 1)) * 2 + h) * (NT * V) + tid * V; };
  auto issue = [&](int row) SO2DR_INLINE {
    if (row < hi0) {
      const int64_t roff = (int64_t)(row - sy0) * a.pitch;
      const int cpb = row_cpb(a.in + roff);  // warp-uniform
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < V; v += VEC)
          issue_vec<T, VEC>(slot(row, h) + v, a.in + roff + xt[h] + v, cpb, xt[h] + v, a.pitch);
    }
    cp_async_commit();
  };
  // steady-state addressing off a running row offset (no 64-bit multiplies):
  // load row = row0 + kRing - 1, store row = row0 - S(R+1)
  int64_t off = (int64_t)(lo0 - sy0) * a.pitch;
  const T* ldb = a.in + (int64_t)(kRing - 1) * a.pitch;
  T* stb = a.out - (int64_t)(S * (R + 1)) * a.pitch;
  auto issue_fast = [&](int row) SO2DR_INLINE {
    if (row < hi0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) issue_inrow<V * 4>(slot(row, h), ldb + off + xt[h]);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < kRing - 1; ++d) issue(lo0 + d);

  auto passthru = [&](int row, int x) SO2DR_INLINE -> T {
    if (x < 0 || x >= a.cols) return T(0);
    return __ldg(a.in + (int64_t)(row - sy0) * a.pitch + x);
  };

  auto body = [&](auto phase_tag, auto fast_tag, int it) SO2DR_INLINE {
    constexpr int PH = decltype(phase_tag)::value;
    constexpr bool FAST = decltype(fast_tag)::value;
    const int row0 = lo0 + it;
#pragma unroll
    for (int u = S; u >= 1; --u) {
      const int A = row0 - u - (u - 1) * R;  // row consumed by stage u
      const int Erow = A - R;                // row emitted by stage u
      const bool consume = FAST || (A >= lo[u - 1] && A < hi[u - 1]);
      const bool emit = FAST || (Erow >= lo[u] && Erow < hi[u]);

      if (u == 1) {
        // stage 1: scalar FFMAs on the loaded A / B vectors into the halves of
        // the pair accumulators (same canonical chain per point)
        float ha[R + V + R], hb[R + V + R];
#pragma unroll
        for (int k = 0; k < V; ++k) {
          ha[R + k] = c0a[k];
          hb[R + k] = c0b[k];
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
          ha[j] = __shfl_up_sync(0xffffffffu, c0a[V - R + j], 1);
          hb[j] = __shfl_up_sync(0xffffffffu, c0b[V - R + j], 1);
          ha[R + V + j] = __shfl_down_sync(0xffffffffu, c0a[j], 1);
          hb[R + V + j] = __shfl_down_sync(0xffffffffu, c0b[j], 1);
        }
        if (consume) {
#pragma unroll
          for (int m = 0; m < E; ++m) {
            const int dy = m - R;
            const int sl = (PH - m + 2 * E) % E;
#pragma unroll
            for (int k = 0; k < V; ++k) {
              float xa = (m == 0) ? 0.f : lo_of(ap[0][sl][k]);
              float xb = (m == 0) ? 0.f : hi_of(ap[0][sl][k]);
              if constexpr (KIND == KBOX) {
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                  const float w = a.w[(dy + R) * E + dx + R];
                  xa = __fmaf_rn(w, ha[R + k + dx], xa);
                  xb = __fmaf_rn(w, hb[R + k + dx], xb);
                }
              } else if (dy != 0) {
                const float w = a.w[(dy + R) * E + R];
                xa = __fmaf_rn(w, ha[R + k], xa);
                xb = __fmaf_rn(w, hb[R + k], xb);
              } else {
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                  const float w = a.w[R * E + dx + R];
                  xa = __fmaf_rn(w, ha[R + k + dx], xa);
                  xb = __fmaf_rn(w, hb[R + k + dx], xb);
                }
              }
              ap[0][sl][k] = pack2(xa, xb);
            }
          }
        }
      } else {
      uint64_t in[V];
#pragma unroll
      for (int k = 0; k < V; ++k) in[k] = ap[u >= 2 ? u - 2 : 0][PH][k];
      // operand pairs: op[i] = (A s_i, B s_i), s_i = cell i-R (halo for i < R or i >= R+V);
      // lanes 0 / 31 receive their own values: strip-edge garbage, never stored
      uint64_t op[V + 2 * R];
#pragma unroll
      for (int k = 0; k < V; ++k) op[R + k] = in[k];
      // 64-bit shuffles move a whole (A, B) pair: the two SHFLs land in an
      // aligned register pair, ready as an FFMA2 operand
#pragma unroll
      for (int j = 0; j < R; ++j) {
        op[j] = __shfl_up_sync(0xffffffffu, in[V - R + j], 1);
        op[R + V + j] = __shfl_down_sync(0xffffffffu, in[j], 1);
      }

      if (consume) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
          const int dy = m - R;                 // the consumed row contributes at dy
          const int sl = (PH - m + 2 * E) % E;  // slot of output row A - dy
#pragma unroll
          for (int k = 0; k < V; ++k) {
            uint64_t x = (m == 0) ? 0ull : ap[u - 1][sl][k];
            if constexpr (KIND == KBOX) {
#pragma unroll
              for (int dx = -R; dx <= R; ++dx) x = fma2p(a.w[(dy + R) * E + dx + R], op[R + k + dx], x);
            } else if (dy != 0) {
              x = fma2p(a.w[(dy + R) * E + R], op[R + k], x);
            } else {
#pragma unroll
              for (int dx = -R; dx <= R; ++dx) x = fma2p(a.w[R * E + dx + R], op[R + k + dx], x);
            }
            ap[u - 1][sl][k] = x;
          }
        }
      }
      }
      if (emit) {
        constexpr int se = (PH - 2 * R + 2 * E) % E;  // slot of row A - R
        if constexpr (!FAST) {
          const bool ring_row = Erow < a.iy0 || Erow >= a.iy1;
          if (ring_row || (ringmask[0] | ringmask[1])) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
              float va = lo_of(ap[u - 1][se][k]), vb = hi_of(ap[u - 1][se][k]);
              if (ring_row || (ringmask[0] & (1u << k))) va = passthru(Erow, xt[0] + k);
              if (ring_row || (ringmask[1] & (1u << k))) vb = passthru(Erow, xt[1] + k);
              ap[u - 1][se][k] = pack2(va, vb);
            }
          }
        }
        if (u == S) {
          T* da = stb + off + xt[0];  // row Erow = row0 - S(R+1)
          T* db = stb + off + xt[1];
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if (smask[0] & (1u << k)) da[k] = lo_of(ap[u - 1][se][k]);
            if (smask[1] & (1u << k)) db[k] = hi_of(ap[u - 1][se][k]);
          }
        }
      }
    }
    // stage 0: row lo0 + it arrives from the cp.async ring
    if constexpr (FAST)
      issue_fast(row0 + kRing - 1);
    else
      issue(row0 + kRing - 1);
    cp_async_wait<kRing - 1>();
    off += a.pitch;
    if (FAST || row0 < hi0) {
      const T* sa = slot(row0, 0);
      const T* sb = slot(row0, 1);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        c0a[k] = sa[k];
        c0b[k] = sb[k];
      }
    }
  };

  // steady-state window (identical derivation to k1_item_pk)
  int f_lo = 0, f_hi = hi0 - lo0;
#pragma unroll
  for (int u = 1; u <= S; ++u) {
    const int c = lo0 - u - (u - 1) * R;
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
  const int fl = (f_lo + E - 1) / E * E;
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

// Persistent warps pulling (strip pair, segment) items; pairs holding a ring
// strip (the first nlp pairs) are handed out first (longest items first).
template <int R, int S, int KIND, int V, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k1_stencil2d_p2(const K1Args2D<float> a) {
  extern __shared__ __align__(16) float ring[];
  const int lane = threadIdx.x & 31;
  const int np = (a.warps_x + 1) / 2;
  const int nlp = a.nl > a.nr ? a.nl : a.nr;
  const int total = np * a.nseg;
  for (;;) {
    int item = 0;
    if (lane == 0) item = static_cast<int>(atomicAdd(a.counter, 1u));
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= total) break;
    int q, sg;
    if (nlp >= np) {
      sg = item / np;
      q = item - sg * np;
    } else if (item < nlp * a.nseg) {
      sg = item / nlp;
      q = item - sg * nlp;
    } else {
      const int inner = np - nlp, i = item - nlp * a.nseg;
      sg = i / inner;
      q = nlp + (i - sg * inner);
    }
    k1_item_p2<R, S, KIND, V, NT>(a, q, sg, ring);
  }
}

}  // namespace so2dr_dev

// k1_3d.cu -- K1 for 3D grids: the k-step temporal-blocked star/box kernel
// streamed along z (the chunking dimension), sm_100a.
//
// Same contract as the 2D K1 (one reference fused_kernel call, generalised to
// 3D, see SURVEY 8(a) a16 and DESIGN.md 4): planes [y0, y1) of the write buffer
// receive the state after S steps; every in-plane cell of those planes is
// written; cells outside the interior (ring planes / ring rows / ring columns)
// pass through. Per-point arithmetic: +0 then one FMA per tap in canonical
// (dz, dy, dx) ascending order (star: on-axis taps only) -- the restated oracle
// (oracle/so2dr_oracle.c) and, for dz != 0 weights zero, the 2D reference.
//
// Design:
//  * A CTA owns an x-y tile of (32*V) x (NW*VY) cells: lane l holds V
//    consecutive x cells, warp w holds VY consecutive rows. It streams the
//    tile's planes (segment +- R*S warm-up planes) from HBM once; the outer
//    R*S cells of the tile on each side are the recomputed temporal-blocking
//    halo.
//  * S time steps = S pipeline stages; stage u consumes the plane stage u-1
//    emitted one iteration earlier and keeps 2R+1 partial-accumulator planes,
//    so each point receives its taps in canonical (dz, dy, dx) order.
//  * x neighbours: warp shuffles. y neighbours in other warps: each stage
//    publishes its warp's top/bottom R rows to shared memory (double-buffered
//    by iteration parity, one __syncthreads per iteration).
//  * Input planes: cp.async into a per-thread ring, read back by the issuing
//    thread only.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <utility>

#include "k1_2d.cuh"  // fma_rn, cp_async helpers
#include "k1_launch.h"

namespace so2dr_dev {

template <typename T>
struct K1Args3D {
  const T* in;
  T* out;
  int64_t pitch;         // elements per storage row
  int64_t plane_stride;  // elements per plane (= p * pitch)
  int base, planes;      // storage planes [base, base+planes)
  int p;                 // padded edge (rows per plane, cols per row)
  int z0, z1;            // output planes
  int iz0, iz1;          // interior planes
  int i0, i1;            // in-plane interior [i0, i1) for y and x
  int seg;               // output planes per CTA
  int tile_x, tile_y;    // valid output cells per CTA along x / y
  int xorg, yorg;        // origin of CTA (0,0)'s thread cell (aligned)
  int cpb;               // cp.async piece bytes (largest of 16/8/4 dividing the pitch)
  T w[125];              // (2R+1)^3 canonical weights
};

template <typename T, int R, int S, int KIND, int V, int VY, int NT>
__global__ void __launch_bounds__(NT, 1) k1_stencil3d(const K1Args3D<T> a) {
  constexpr int E = 2 * R + 1, H = R * S, NW = NT / 32;
  constexpr int RING = 4;
  constexpr int CPB = (V * (int)sizeof(T)) >= 16 ? 16 : V * (int)sizeof(T);
  constexpr int VEC = CPB / (int)sizeof(T);
  static_assert(R <= V && R <= VY, "halo must come from the neighbouring thread only");

  // dynamic shared memory: input ring [RING][VY][NT*V], then the y-halo
  // exchange [parity][stage][warp+1][top/bottom][R][32*V] (+2 guard warps)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Ring = T[RING][VY][NT * V];
  using YEdge = T[2][S][NW + 2][2][R][32 * V];
  Ring& ring = *reinterpret_cast<Ring*>(smem_raw);
  YEdge& yedge = *reinterpret_cast<YEdge*>(smem_raw + sizeof(Ring));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cx0 = a.xorg + blockIdx.x * a.tile_x;  // x of lane 0 cell 0
  const int cy0 = a.yorg + blockIdx.y * a.tile_y;  // y of warp 0 row 0
  const int xt = cx0 + lane * V;
  const int yt = cy0 + warp * VY;
  const int OZ0 = a.z0 + blockIdx.z * a.seg;
  const int OZ1 = min(OZ0 + a.seg, a.z1);
  const int sz0 = a.base, sz1 = a.base + a.planes;
  const int lo0 = max(OZ0 - H, sz0), hi0 = min(OZ1 + H, sz1);
  const int n_iter = OZ1 - lo0 + S * (R + 1);
  // valid output window of this CTA
  const int OX0 = max(cx0 + H, 0), OX1 = min(cx0 + H + a.tile_x, a.p);
  const int OY0 = max(cy0 + H, 0), OY1 = min(cy0 + H + a.tile_y, a.p);

  int lo[S + 1], hi[S + 1];
#pragma unroll
  for (int u = 0; u <= S; ++u) {
    lo[u] = max(OZ0 - R * (S - u), sz0);
    hi[u] = min(OZ1 + R * (S - u), sz1);
  }

  // per-cell masks over the thread's VY x V cells (bit j*V+k)
  unsigned ringmask = 0, smask = 0, inmask = 0;
#pragma unroll
  for (int j = 0; j < VY; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int x = xt + k, y = yt + j;
      const unsigned bit = 1u << (j * V + k);
      if (x < a.i0 || x >= a.i1 || y < a.i0 || y >= a.i1) ringmask |= bit;
      if (x >= OX0 && x < OX1 && y >= OY0 && y < OY1) smask |= bit;
      if (x >= 0 && x < a.p && y >= 0 && y < a.p) inmask |= bit;
    }

  for (int i = tid; i < 2 * S * (NW + 2) * 2 * R * 32 * V; i += NT)
    (&yedge[0][0][0][0][0][0])[i] = T(0);

  T cur[S][VY][V];
  T acc[S][E][VY][V];
#pragma unroll
  for (int u = 0; u < S; ++u)
#pragma unroll
    for (int j = 0; j < VY; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) cur[u][j][k] = T(0);

  auto issue = [&](int plane) SO2DR_INLINE {
    const bool ok = plane < hi0;
    const T* src = a.in + (int64_t)(plane - sz0) * a.plane_stride;
#pragma unroll
    for (int j = 0; j < VY; ++j) {
      const int y = yt + j;
      const bool rok = ok && y >= 0 && y < a.p;
#pragma unroll
      for (int v = 0; v < V; v += VEC)
        if (rok)
          issue_vec<T, VEC>(&ring[plane & (RING - 1)][j][tid * V + v], src + (int64_t)y * a.pitch + xt + v,
                            a.cpb, xt + v, a.pitch);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < RING - 1; ++d) issue(lo0 + d);
  __syncthreads();

  // steady-state addressing off a running plane offset (poff = (row0 - sz0) *
  // plane_stride, advanced once per iteration): load plane row0 + RING - 1,
  // store plane row0 - S(R+1); the thread's (y, x) part is loop-invariant
  int64_t poff = (int64_t)(lo0 - sz0) * a.plane_stride;
  const T* ld_thr = a.in + (int64_t)(RING - 1) * a.plane_stride + (int64_t)yt * a.pitch + xt;
  T* st_thr = a.out - (int64_t)(S * (R + 1)) * a.plane_stride + (int64_t)yt * a.pitch + xt;
  auto issue_fast = [&](int plane) SO2DR_INLINE {
    if (plane < hi0) {
#pragma unroll
      for (int j = 0; j < VY; ++j)
        issue_inrow<V * (int)sizeof(T)>(&ring[plane & (RING - 1)][j][tid * V], ld_thr + poff + (int64_t)j * a.pitch);
    }
    cp_async_commit();
  };

  auto passthru = [&](int plane, int j, int k) SO2DR_INLINE -> T {
    const int x = xt + k, y = yt + j;
    if (x < 0 || x >= a.p || y < 0 || y >= a.p) return T(0);
    return __ldg(a.in + (int64_t)(plane - sz0) * a.plane_stride + (int64_t)y * a.pitch + x);
  };

  auto publish_edges = [&](int par, int u, const T (&v)[VY][V]) {
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        yedge[par][u][warp + 1][0][j][lane * V + k] = v[j][k];
        yedge[par][u][warp + 1][1][j][lane * V + k] = v[VY - R + j][k];
      }
  };

  // FAST = steady state of a CTA whose whole tile is interior: every stage
  // consumes and emits interior planes, no ring pass-through, no grid-edge
  // masking -- all range checks compile away (as in the 2D K1).
  auto body = [&](auto phase_tag, auto fast_tag, int it) SO2DR_INLINE {
    constexpr int PH = decltype(phase_tag)::value;
    constexpr bool FAST = decltype(fast_tag)::value;
    const int par = it & 1, ppar = par ^ 1;
    const int row0 = lo0 + it;
#pragma unroll
    for (int u = S; u >= 1; --u) {
      const int A = row0 - u - (u - 1) * R;
      const int Ez = A - R;
      const bool consume = FAST || (A >= lo[u - 1] && A < hi[u - 1]);
      const bool emit = FAST || (Ez >= lo[u] && Ez < hi[u]);

      // neighbourhood of the consumed plane: rows yt-R .. yt+VY-1+R,
      // cols xt-R .. xt+V-1+R
      T nb[VY + 2 * R][V + 2 * R];
#pragma unroll
      for (int j = 0; j < VY; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) nb[R + j][R + k] = cur[u - 1][j][k];
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) {
          nb[j][R + k] = yedge[ppar][u - 1][warp][1][j][lane * V + k];          // warp above, bottom rows
          nb[R + VY + j][R + k] = yedge[ppar][u - 1][warp + 2][0][j][lane * V + k];  // warp below, top rows
        }
#pragma unroll
      for (int j = 0; j < VY + 2 * R; ++j)
#pragma unroll
        for (int q = 0; q < R; ++q) {
          nb[j][q] = __shfl_up_sync(0xffffffffu, nb[j][V + q], 1);
          nb[j][R + V + q] = __shfl_down_sync(0xffffffffu, nb[j][R + q], 1);
        }

      if (consume) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
          const int dz = m - R;
          const int sl = (PH - m + 2 * E) % E;
#pragma unroll
          for (int j = 0; j < VY; ++j)
#pragma unroll
            for (int k = 0; k < V; ++k) {
              T x = (m == 0) ? T(0) : acc[u - 1][sl][j][k];
              if constexpr (KIND == KBOX) {
#pragma unroll
                for (int dy = -R; dy <= R; ++dy)
#pragma unroll
                  for (int dx = -R; dx <= R; ++dx)
                    x = fma_rn(a.w[((dz + R) * E + dy + R) * E + dx + R], nb[R + j + dy][R + k + dx], x);
              } else if (dz != 0) {
                x = fma_rn(a.w[((dz + R) * E + R) * E + R], nb[R + j][R + k], x);
              } else {
#pragma unroll
                for (int dy = -R; dy < 0; ++dy)
                  x = fma_rn(a.w[(R * E + dy + R) * E + R], nb[R + j + dy][R + k], x);
#pragma unroll
                for (int dx = -R; dx <= R; ++dx)
                  x = fma_rn(a.w[(R * E + R) * E + dx + R], nb[R + j][R + k + dx], x);
#pragma unroll
                for (int dy = 1; dy <= R; ++dy)
                  x = fma_rn(a.w[(R * E + dy + R) * E + R], nb[R + j + dy][R + k], x);
              }
              acc[u - 1][sl][j][k] = x;
            }
        }
      }

      if (emit) {
        constexpr int se = (PH - 2 * R + 2 * E) % E;
        T outv[VY][V];
        const bool ring_plane = !FAST && (Ez < a.iz0 || Ez >= a.iz1);
#pragma unroll
        for (int j = 0; j < VY; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k) {
            outv[j][k] = acc[u - 1][se][j][k];
            if constexpr (!FAST)
              if (ring_plane || (ringmask & (1u << (j * V + k)))) outv[j][k] = passthru(Ez, j, k);
          }
        if (u == S) {
          if constexpr (FAST) {
            T* dst = st_thr + poff;
#pragma unroll
            for (int j = 0; j < VY; ++j)
#pragma unroll
              for (int k = 0; k < V; ++k)
                if (smask & (1u << (j * V + k))) dst[(int64_t)j * a.pitch + k] = outv[j][k];
          } else {
            T* dst = a.out + (int64_t)(Ez - sz0) * a.plane_stride;
#pragma unroll
            for (int j = 0; j < VY; ++j)
#pragma unroll
              for (int k = 0; k < V; ++k)
                if (smask & (1u << (j * V + k))) dst[(int64_t)(yt + j) * a.pitch + xt + k] = outv[j][k];
          }
        } else {
#pragma unroll
          for (int j = 0; j < VY; ++j)
#pragma unroll
            for (int k = 0; k < V; ++k) cur[u][j][k] = outv[j][k];
          publish_edges(par, u, outv);
        }
      }
    }

    // stage 0
    if constexpr (FAST)
      issue_fast(row0 + RING - 1);
    else
      issue(row0 + RING - 1);
    cp_async_wait<RING - 1>();
    if (FAST || row0 < hi0) {
#pragma unroll
      for (int j = 0; j < VY; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k)
          cur[0][j][k] = (FAST || (inmask & (1u << (j * V + k)))) ? ring[row0 & (RING - 1)][j][tid * V + k] : T(0);
      publish_edges(par, 0, cur[0]);
    }
    poff += a.plane_stride;
    __syncthreads();
  };

  // steady-state window [f_lo, f_hi) of iterations (same derivation as 2D);
  // CTA-uniform, so the one barrier per iteration stays uniform
  int f_lo = 0, f_hi = hi0 - lo0;
#pragma unroll
  for (int u = 1; u <= S; ++u) {
    const int c = lo0 - u - (u - 1) * R;
    f_lo = max(f_lo, lo[u - 1] - c);
    f_hi = min(f_hi, hi[u - 1] - c);
    f_lo = max(f_lo, max(lo[u], a.iz0) + R - c);
    f_hi = min(f_hi, min(hi[u], a.iz1) + R - c);
  }
  const bool tile_interior = cx0 >= a.i0 && cx0 + 32 * V <= a.i1 && cy0 >= a.i0 && cy0 + NW * VY <= a.i1;
  if (!tile_interior) f_hi = f_lo;

  int it = 0;
  auto run_general = [&](int stop) SO2DR_INLINE {
    while (it < stop) {
      [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
        ((it < stop ? (body(std::integral_constant<int, Ps>{}, std::false_type{}, it), ++it, void()) : void()),
         ...);
      }(std::make_integer_sequence<int, E>{});
    }
  };
  // (the radius-2 box's 125-tap pipeline has no register room for a second
  // copy of the loop: it runs the general path only, no spill)
  if constexpr (!(KIND == KBOX && R >= 2)) {
    const int fl = (f_lo + E - 1) / E * E;
    if (f_hi - fl >= E) {
      run_general(fl);
      while (it + E <= f_hi) {
        [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
          ((body(std::integral_constant<int, Ps>{}, std::true_type{}, it), ++it), ...);
        }(std::make_integer_sequence<int, E>{});
      }
    }
  }
  run_general(n_iter);
  cp_async_wait<0>();
}

namespace {

inline int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Tile shape of the 3D K1 per thread (V x VY cells) and CTA size. Default
// 2x2 cells, 512 threads. SO2DR_K1_3D=42 / 44 select 4x2 / 4x4 cells on 256
// threads for fp32 radius 1 (experiments: more FMAs per shuffle/LDS/barrier).
inline int k1_3d_shape() {
  static int v = [] {
    const char* e = std::getenv("SO2DR_K1_3D");
    return e ? std::atoi(e) : 22;
  }();
  return v;
}

template <typename T, int R, int S, int KIND, int V = 2, int VY = 2,
          int NT = (sizeof(T) == 8 && R == 2) ? 256 : 512>
cudaError_t launch3(const K1Launch& L, cudaStream_t stream) {
  // 512 threads cap registers at 128; the fp64 radius-2 box needs more (a spill
  // otherwise), so it runs 256-thread CTAs
  constexpr int NW = NT / 32, H = R * S;
  constexpr size_t smem = sizeof(T) * (4 * VY * NT * V + 2 * S * (NW + 2) * 2 * R * 32 * V);
  static_assert(smem <= 227 * 1024, "3D K1 shared memory");
  auto kern = k1_stencil3d<T, R, S, KIND, V, VY, NT>;
  static bool attr_done = false;
  if (!attr_done) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  constexpr int CPB = (V * (int)sizeof(T)) >= 16 ? 16 : V * (int)sizeof(T);
  constexpr int VEC = CPB / (int)sizeof(T);
  K1Args3D<T> a;
  a.in = static_cast<const T*>(L.in);
  a.out = static_cast<T*>(L.out);
  a.pitch = L.pitch;
  {
    const int64_t pb = L.pitch * static_cast<int64_t>(sizeof(T));
    a.cpb = pb % 16 == 0 ? 16 : pb % 8 == 0 ? 8 : 4;
  }
  a.p = L.cols;
  a.plane_stride = static_cast<int64_t>(L.plane_rows) * L.pitch;
  a.base = L.base;
  a.planes = L.rows;
  a.z0 = L.y0;
  a.z1 = L.y1;
  a.iz0 = L.iy0;
  a.iz1 = L.iy1;
  a.i0 = L.ix0;
  a.i1 = L.ix1;
  constexpr int E = 2 * R + 1;
  for (int i = 0; i < 125; ++i) a.w[i] = T(0);
  for (int i = 0; i < E * E * E; ++i) a.w[i] = static_cast<T>(L.w[i]);
  a.tile_x = ((32 * V - 2 * H) / VEC) * VEC;
  a.tile_y = NW * VY - 2 * H;
  if (a.tile_x <= 0 || a.tile_y <= 0) return cudaErrorInvalidValue;
  a.xorg = fdiv(-H, VEC) * VEC;
  a.yorg = -H;
  const int nx = (a.p - (a.xorg + H) + a.tile_x - 1) / a.tile_x;
  const int ny = (a.p - (a.yorg + H) + a.tile_y - 1) / a.tile_y;
  const int depth = L.y1 - L.y0;
  const int sms = device_sm_count();
  const int min_seg = std::max(16, 4 * (H + S * (R + 1)));
  int nz = std::max(1, (4 * sms + nx * ny - 1) / (nx * ny));
  nz = std::min(nz, std::max(1, depth / min_seg));
  a.seg = (depth + nz - 1) / nz;
  nz = (depth + a.seg - 1) / a.seg;
  dim3 grid(nx, ny, nz);
  kern<<<grid, NT, smem, stream>>>(a);
  return cudaGetLastError();
}

template <typename T>
constexpr int maxs3d(int R) {
  return sizeof(T) == 4 ? (R == 1 ? 4 : 2) : (R == 1 ? 2 : 1);
}

template <typename T, int R, int KIND, int S = 1>
cudaError_t launch3_s(const K1Launch& L, cudaStream_t stream) {
  if constexpr (S > maxs3d<T>(R)) {
    return cudaErrorInvalidValue;
  } else {
    if (L.steps == S) {
      if constexpr (sizeof(T) == 4 && R == 1) {
        if (k1_3d_shape() == 42) return launch3<T, R, S, KIND, 4, 2, 256>(L, stream);
        if constexpr (S <= 2) {
          if (k1_3d_shape() == 44) return launch3<T, R, S, KIND, 4, 4, 256>(L, stream);
        }
      }
      return launch3<T, R, S, KIND>(L, stream);
    }
    return launch3_s<T, R, KIND, S + 1>(L, stream);
  }
}

template <typename T>
cudaError_t launch3_any(const K1Launch& L, cudaStream_t stream) {
  if (L.steps < 1 || !L.w) return cudaErrorInvalidValue;
  if (L.kind == KBOX) {
    if (L.radius == 1) return launch3_s<T, 1, KBOX>(L, stream);
    if (L.radius == 2) return launch3_s<T, 2, KBOX>(L, stream);
  } else if (L.kind == KSTAR) {
    if (L.radius == 1) return launch3_s<T, 1, KSTAR>(L, stream);
    if (L.radius == 2) return launch3_s<T, 2, KSTAR>(L, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_k1_3d_f32(const K1Launch& L, cudaStream_t s) { return launch3_any<float>(L, s); }
cudaError_t launch_k1_3d_f64(const K1Launch& L, cudaStream_t s) { return launch3_any<double>(L, s); }

}  // namespace so2dr_dev

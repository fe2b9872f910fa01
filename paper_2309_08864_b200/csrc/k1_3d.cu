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
#include "k1_segplan.h"

#ifndef SO2DR_K3D_SHAPE  // fp32 radius-1 cells per thread: 22 = 2x2 on 512 threads, 24 = 2x4 on 256
#define SO2DR_K3D_SHAPE 22
#endif

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
  int seg_b, nseg_b;     // z segments: nseg_b big ones of seg_b planes from z0,
  int seg_s, nseg_s;     // then small ones of seg_s (handed out last: k1_plan_segments)
  int tile_x, tile_y;    // valid output cells per CTA along x / y
  int xorg, yorg;        // origin of CTA (0,0)'s thread cell (aligned)
  int cpb;               // cp.async piece bytes (largest of 16/8/4 dividing the pitch)
  int nx, ny;            // tiles along x / y (work items nx*ny*(nseg_b+nseg_s))
  unsigned* counter;     // work-item counter pair (k1_next_counter)
  T w[125];              // (2R+1)^3 canonical weights
};

// One CTA work item (x-y tile, z segment). Every iteration runs the same
// body, including the pipeline fill and drain (as the 2D streaming path,
// k1_2d_stream.cuh): a plane a stage computes from planes outside its light
// cone never reaches a stored plane. Pass-through cells (ring planes / rows /
// columns): after every stage the emitted plane's ring cells are reset to the
// read buffer's value (a CTA-uniform test per plane); tiles that hang over the
// padded grid load with per-element range checks.
template <typename T, int R, int S, int KIND, int V, int VY, int NT, bool EDGE>
__device__ __forceinline__ void k1_tile3d(const K1Args3D<T>& a, int tx, int ty, int OZ0, int OZ1,
                                          unsigned char* smem_raw) {
  constexpr int E = 2 * R + 1, H = R * S, NW = NT / 32;
  constexpr int RING = 4;
  using Ring = T[RING][VY][NT * V];
  using YEdge = T[2][S][NW + 2][2][R][32 * V];
  Ring& ring = *reinterpret_cast<Ring*>(smem_raw);
  YEdge& yedge = *reinterpret_cast<YEdge*>(smem_raw + sizeof(Ring));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cx0 = a.xorg + tx * a.tile_x;  // x of lane 0 cell 0
  const int cy0 = a.yorg + ty * a.tile_y;  // y of warp 0 row 0
  const int xt = cx0 + lane * V;
  const int yt = cy0 + warp * VY;
  const int sz0 = a.base, sz1 = a.base + a.planes;
  const int lo0 = max(OZ0 - H, sz0), hi0 = min(OZ1 + H, sz1);
  const int n_iter = OZ1 - lo0 + S * (R + 1);
  // valid output window of this tile
  const int OX0 = max(cx0 + H, 0), OX1 = min(cx0 + H + a.tile_x, a.p);
  const int OY0 = max(cy0 + H, 0), OY1 = min(cy0 + H + a.tile_y, a.p);

  // per-cell masks over the thread's VY x V cells (bit j*V+k)
  unsigned ringmask = 0, smask = 0, inmask = 0;
#pragma unroll
  for (int j = 0; j < VY; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int x = xt + k, y = yt + j;
      const unsigned bit = 1u << (j * V + k);
      if (x >= 0 && x < a.p && y >= 0 && y < a.p) {
        inmask |= bit;
        if (x < a.i0 || x >= a.i1 || y < a.i0 || y >= a.i1) ringmask |= bit;
      }
      if (x >= OX0 && x < OX1 && y >= OY0 && y < OY1) smask |= bit;
    }
  // every cell of the tile inside the padded grid: loads need no per-element
  // range checks (CTA-uniform)
  // (EDGE = false: the caller checked that the whole tile is interior in x-y)
  const bool xy_inside = !EDGE || (cx0 >= 0 && cx0 + 32 * V <= a.p && cy0 >= 0 && cy0 + NW * VY <= a.p);

  T cur[S][VY][V];
  T acc[S][E][VY][V];
#pragma unroll
  for (int u = 0; u < S; ++u)
#pragma unroll
    for (int j = 0; j < VY; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) cur[u][j][k] = T(0);

  // running plane offset: poff = (lo0 + it - sz0) * plane_stride; loads plane
  // lo0 + it + RING - 1, stores plane lo0 + it - S(R+1); the thread's (y, x)
  // part is loop-invariant
  int64_t poff = (int64_t)(lo0 - sz0) * a.plane_stride;
  const int64_t yx = (int64_t)yt * a.pitch + xt;
  const T* ld_thr = a.in + (int64_t)(RING - 1) * a.plane_stride + yx;
  T* st_thr = a.out - (int64_t)(S * (R + 1)) * a.plane_stride + yx;
  auto issue = [&](int plane, int64_t off) SO2DR_INLINE {
    if (plane < hi0) {
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (EDGE && !xy_inside) {
          const int y = yt + j;
          if (y >= 0 && y < a.p) {
            const T* src = a.in + (int64_t)(plane - sz0) * a.plane_stride + (int64_t)y * a.pitch;
#pragma unroll
            for (int v = 0; v < V; v += (V * (int)sizeof(T) >= 16 ? 16 / (int)sizeof(T) : V)) {
              constexpr int VEC = (V * (int)sizeof(T) >= 16) ? 16 / (int)sizeof(T) : V;
              issue_vec<T, VEC>(&ring[plane & (RING - 1)][j][tid * V + v], src + xt + v, a.cpb, xt + v, a.pitch);
            }
          }
        } else {
          issue_inrow<V * (int)sizeof(T)>(&ring[plane & (RING - 1)][j][tid * V], ld_thr + off + (int64_t)j * a.pitch);
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < RING - 1; ++d) issue(lo0 + d, (int64_t)(d - (RING - 1)) * a.plane_stride + poff);

  // CTA-uniform: does this item own any pass-through cell (ring column/row of
  // the tile, or a ring plane in the z range its stages emit)?
  // Interior tiles (EDGE = false) own no ring column / row: only the ring
  // planes pass through, and every cell of the tile is inside the grid.
  const bool tile_edge = (EDGE && __syncthreads_or(ringmask != 0)) || lo0 - H < a.iz0 || OZ1 + H > a.iz1;
  auto passthru = [&](int plane, T (&v)[VY][V]) SO2DR_INLINE {
    if (plane < sz0 || plane >= sz1) return;
    const bool ring_plane = plane < a.iz0 || plane >= a.iz1;
    if constexpr (!EDGE) {
      if (!ring_plane) return;
      const T* g = a.in + (int64_t)(plane - sz0) * a.plane_stride + yx;
#pragma unroll
      for (int j = 0; j < VY; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) v[j][k] = __ldg(g + (int64_t)j * a.pitch + k);
      return;
    }
    const unsigned m = ring_plane ? inmask : ringmask;
    if (!m) return;
    const T* g = a.in + (int64_t)(plane - sz0) * a.plane_stride + yx;
#pragma unroll
    for (int j = 0; j < VY; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (m & (1u << (j * V + k))) v[j][k] = __ldg(g + (int64_t)j * a.pitch + k);
  };

  auto publish_edges = [&](int par, int u, const T (&v)[VY][V]) SO2DR_INLINE {
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        yedge[par][u][warp + 1][0][j][lane * V + k] = v[j][k];
        yedge[par][u][warp + 1][1][j][lane * V + k] = v[VY - R + j][k];
      }
  };

  // unrolled by 2E: the accumulator slot (it mod E) and the edge-exchange
  // parity (it mod 2) are compile-time in every phase
  auto body = [&](auto phase_tag, int it) SO2DR_INLINE {
    constexpr int PH = decltype(phase_tag)::value % E;
    constexpr int par = decltype(phase_tag)::value & 1, ppar = par ^ 1;
    const int row0 = lo0 + it;
#pragma unroll
    for (int u = S; u >= 1; --u) {
      const int Ez = row0 - u - (u - 1) * R - R;  // plane emitted by stage u

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
          nb[j][R + k] = yedge[ppar][u - 1][warp][1][j][lane * V + k];              // warp above, bottom rows
          nb[R + VY + j][R + k] = yedge[ppar][u - 1][warp + 2][0][j][lane * V + k];  // warp below, top rows
        }
#pragma unroll
      for (int j = 0; j < VY + 2 * R; ++j)
#pragma unroll
        for (int q = 0; q < R; ++q) {
          nb[j][q] = __shfl_up_sync(0xffffffffu, nb[j][V + q], 1);
          nb[j][R + V + q] = __shfl_down_sync(0xffffffffu, nb[j][R + q], 1);
        }

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

      constexpr int se = (PH - 2 * R + 2 * E) % E;
      T outv[VY][V];
#pragma unroll
      for (int j = 0; j < VY; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) outv[j][k] = acc[u - 1][se][j][k];
      if (tile_edge) passthru(Ez, outv);
      if (u == S) {
        if (Ez >= OZ0 && Ez < OZ1) {
          T* dst = st_thr + poff;
#pragma unroll
          for (int j = 0; j < VY; ++j)
#pragma unroll
            for (int k = 0; k < V; ++k)
              if (smask & (1u << (j * V + k))) dst[(int64_t)j * a.pitch + k] = outv[j][k];
        }
      } else {
#pragma unroll
        for (int j = 0; j < VY; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k) cur[u][j][k] = outv[j][k];
        publish_edges(par, u, outv);
      }
    }

    // stage 0
    issue(row0 + RING - 1, poff);
    cp_async_wait<RING - 1>();
#pragma unroll
    for (int j = 0; j < VY; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
        cur[0][j][k] = ring[row0 & (RING - 1)][j][tid * V + k];  // (cells off the grid: unread stale values, outside every stored cone)
    publish_edges(par, 0, cur[0]);
    poff += a.plane_stride;
    __syncthreads();
  };

  int it = 0;
  while (it < n_iter) {
    [&]<int... Ps>(std::integer_sequence<int, Ps...>) {
      ((it < n_iter ? (body(std::integral_constant<int, Ps>{}, it), ++it, void()) : void()), ...);
    }(std::make_integer_sequence<int, 2 * E>{});
  }
  cp_async_wait<0>();
}

// Persistent CTAs with dynamic tile scheduling (one wave; no partial last
// wave): every CTA pulls (tile, z segment) items from a per-stream counter and
// re-arms it at the end (k1_next_counter).
template <typename T, int R, int S, int KIND, int V, int VY, int NT>
__global__ void __launch_bounds__(NT, 1) k1_stencil3d(const K1Args3D<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NW = NT / 32;
  __shared__ int s_item;
  using YEdge = T[2][S][NW + 2][2][R][32 * V];
  YEdge& yedge = *reinterpret_cast<YEdge*>(smem_raw + sizeof(T[4][VY][NT * V]));
  // the guard warps' edge rows (above warp 0 / below the last warp) are never
  // written: zero them once (finite garbage for the tile's outer halo)
  for (int i = threadIdx.x; i < 2 * S * (NW + 2) * 2 * R * 32 * V; i += NT) (&yedge[0][0][0][0][0][0])[i] = T(0);
  const int tiles = a.nx * a.ny;
  const int total = tiles * (a.nseg_b + a.nseg_s);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = static_cast<int>(atomicAdd(a.counter, 1u));
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    // (the k1_seg_decode order with no edge units, written out: the shared
    // helper costs this kernel an 8-byte stack frame at its 128-register cap)
    int tz = item / tiles;
    const int rem = item - tz * tiles;
    const int ty = rem / a.nx, tx = rem - ty * a.nx;
    int oz0;
    if (tz < a.nseg_b) {
      oz0 = a.z0 + tz * a.seg_b;
    } else {
      tz -= a.nseg_b;
      oz0 = a.z0 + a.nseg_b * a.seg_b + tz * a.seg_s;
    }
    const int oz1 = min(oz0 + (item < tiles * a.nseg_b ? a.seg_b : a.seg_s), a.z1);
    // x-y interior tile: no ring cell, no cell off the grid (CTA-uniform)
    const int cx0 = a.xorg + tx * a.tile_x, cy0 = a.yorg + ty * a.tile_y;
    // One variant only where two inlined pipelines do not fit: fp64 radius 2
    // (the state spills) and the long box bodies (> 64 fmas per cell and
    // iteration: the doubled loop code misses the instruction cache -- box3d1r
    // k=4 measured -11% with both, k=2 +9%)
    constexpr int kTaps = KIND == KBOX ? (2 * R + 1) * (2 * R + 1) * (2 * R + 1) : 6 * R + 1;
    constexpr bool kInnerVariant = !(sizeof(T) == 8 && R == 2) && S * kTaps <= 64;
    if (kInnerVariant && cx0 >= a.i0 && cx0 + 32 * V <= a.i1 && cy0 >= a.i0 && cy0 + NW * VY <= a.i1)
      k1_tile3d<T, R, S, KIND, V, VY, NT, false>(a, tx, ty, oz0, oz1, smem_raw);
    else
      k1_tile3d<T, R, S, KIND, V, VY, NT, true>(a, tx, ty, oz0, oz1, smem_raw);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.counter + 1, 1u) == gridDim.x - 1) {
      a.counter[0] = 0u;
      a.counter[1] = 0u;
      __threadfence();
    }
  }
}

namespace {

inline int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

template <typename T, int R, int S, int KIND, int V = 2, int VY = 4, int NT = 256>
cudaError_t launch3(const K1Launch& L, cudaStream_t stream) {
  // 2x4 cells per thread on 256 threads: the same 64x32 tile as 2x2 on 512,
  // fewer shuffles / edge rows per cell, and room (255 registers) for both
  // the inner and the edge variant of the pipeline without spills
  constexpr int NW = NT / 32, H = R * S;
  constexpr size_t smem = sizeof(T) * (4 * VY * NT * V + 2 * S * (NW + 2) * 2 * R * 32 * V);
  static_assert(smem <= 227 * 1024, "3D K1 shared memory");
  auto kern = k1_stencil3d<T, R, S, KIND, V, VY, NT>;
  static bool attr_done[64] = {};
  {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr_done[dev]) {  // per device: the attribute applies to the current device only
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_done[dev] = true;
    }
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
  a.nx = nx;
  a.ny = ny;
  static int occ_by_dev[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  int occ = occ_by_dev[dev];
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem) != cudaSuccess || occ < 1) occ = 1;
    occ_by_dev[dev] = occ;
  }
  // z segmentation: guided plan over the persistent CTAs (big segments, then
  // small ones that even out the finish times); an item recomputes its H
  // warm-up planes and the S(R+1)-plane pipeline fill
  const int ov = H + S * (R + 1) + 4;
  const int min_seg_u = std::max(16, 4 * (H + S * (R + 1)));  // r02-mid: ~8 items per SM
  static const int ips = [] {  // uniform z items per SM (SO2DR_K3D_IPS: experiments)
    const char* e = std::getenv("SO2DR_K3D_IPS");
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  int nz_u = std::max(1, (ips * sms + nx * ny - 1) / (nx * ny));
  nz_u = std::min(nz_u, std::max(1, depth / min_seg_u));
  const int seg_u = std::max(1, (depth + nz_u - 1) / nz_u);
  const K1SegPlan sp = k1_plan_segments(depth, nx * ny, 0, (int64_t)sms * occ, ov, 1.0, std::max(8, 2 * ov), seg_u);
  a.seg_b = sp.seg_b, a.nseg_b = sp.nseg_b;
  a.seg_s = sp.seg_s, a.nseg_s = sp.nseg_s;
  const int64_t items = (int64_t)nx * ny * (a.nseg_b + a.nseg_s);
  a.counter = k1_next_counter(stream);
  if (!a.counter) return cudaErrorUnknown;
  const int ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, items));
  kern<<<ctas, NT, smem, stream>>>(a);
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
      // radius 2 box (125 taps) and fp64 radius 2: 2x2 cells per thread (the
      // 2x4 pipeline spills)
      if constexpr (R == 2 && (KIND == KBOX || sizeof(T) == 8)) return launch3<T, R, S, KIND, 2, 2, 256>(L, stream);
      else if constexpr (sizeof(T) == 4 && R == 1 && SO2DR_K3D_SHAPE == 22) return launch3<T, R, S, KIND, 2, 2, 512>(L, stream);
      else return launch3<T, R, S, KIND>(L, stream);
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

/*
 * so2dr_oracle.c -- CPU restatement of the SO2DR reference arithmetic.
 * TEST INFRASTRUCTURE ONLY (see so2dr_oracle.h). Compile with
 * -ffp-contract=off: every multiply-add below is an explicit fma()/fmaf()
 * and every other operation must round on its own, exactly as the reference
 * is built (proj/CMakeLists.txt:20).
 */
#include "so2dr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* proj/src/stencil.cpp:92-97 splitmix64 finaliser */
static uint64_t orc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* proj/src/stencil.cpp:99-106: counter = (u32 y << 32) | u32 x, value =
 * top 24 bits of mix64(seed ^ mix64(counter)) scaled by 2^-24. */
float orc_cell_value(uint64_t seed, int y, int x) {
  const uint64_t counter = ((uint64_t)(uint32_t)y << 32) | (uint64_t)(uint32_t)x;
  const uint64_t h = orc_mix64(seed ^ orc_mix64(counter));
  return (float)(h >> 40) * 0x1p-24f;
}

float orc_cell_value3(uint64_t seed, int z, int y, int x) {
  return orc_cell_value(seed ^ ((uint64_t)(uint32_t)z * 0x9E3779B97F4A7C15ULL), y, x);
}

void orc_init_f32(float* g, int dim, int sz, int r, uint64_t seed) {
  const int p = sz + 2 * r;
  const int pz = dim == 3 ? p : 1;
  size_t i = 0;
  for (int z = 0; z < pz; ++z)
    for (int y = 0; y < p; ++y)
      for (int x = 0; x < p; ++x)
        g[i++] = dim == 3 ? orc_cell_value3(seed, z, y, x) : orc_cell_value(seed, y, x);
}

void orc_init_f64(double* g, int dim, int sz, int r, uint64_t seed) {
  const int p = sz + 2 * r;
  const int pz = dim == 3 ? p : 1;
  size_t i = 0;
  for (int z = 0; z < pz; ++z)
    for (int y = 0; y < p; ++y)
      for (int x = 0; x < p; ++x)
        g[i++] = (double)(dim == 3 ? orc_cell_value3(seed, z, y, x) : orc_cell_value(seed, y, x));
}

/* init_grid values of the box [z0,z0+nz) x [y0,y0+ny) x [x0,x0+nx) of the
 * padded grid (dim 2: z ignored, nz = 1). */
void orc_init_block_f32(float* g, int dim, int z0, int y0, int x0, int nz, int ny, int nx, uint64_t seed) {
  size_t i = 0;
  for (int z = z0; z < z0 + nz; ++z)
    for (int y = y0; y < y0 + ny; ++y)
      for (int x = x0; x < x0 + nx; ++x)
        g[i++] = dim == 3 ? orc_cell_value3(seed, z, y, x) : orc_cell_value(seed, y, x);
}

void orc_init_block_f64(double* g, int dim, int z0, int y0, int x0, int nz, int ny, int nx, uint64_t seed) {
  size_t i = 0;
  for (int z = z0; z < z0 + nz; ++z)
    for (int y = y0; y < y0 + ny; ++y)
      for (int x = x0; x < x0 + nx; ++x)
        g[i++] = (double)(dim == 3 ? orc_cell_value3(seed, z, y, x) : orc_cell_value(seed, y, x));
}

/* The per-point rule, written once per element type. Box: accumulator starts
 * at +0 and takes one fused multiply-add per tap in canonical order
 * (proj/src/stencil.cpp:137-143; dz outermost for 3D). Star: the same chain
 * restricted to on-axis taps (a box with zero off-axis weights gives the same
 * bits for finite data because fma(0, v, acc) == acc when acc != -0, and the
 * chain never produces -0 from a +0 start). Gradient: the pinned expression of
 * proj/src/stencil.cpp:122-135, no contraction. */
#define ORC_DEFINE_STEP(SUFFIX, T, FMA)                                              \
  static T orc_point_##SUFFIX(const T* in, size_t c, size_t sy, size_t sz_,         \
                              int r, int dim, int kind, const double* w) {           \
    if (kind == ORC_GRADIENT) {                                                     \
      const T v = in[c];                                                             \
      const T dn = in[c - sy] - v;                                                   \
      const T ds = in[c + sy] - v;                                                   \
      const T de = in[c + 1] - v;                                                    \
      const T dw = in[c - 1] - v;                                                    \
      const T sum = ((dn + ds) + de) + dw;                                           \
      const T q = (T)0.25 * sum;                                                     \
      return v + q;                                                                  \
    }                                                                                \
    T acc = (T)0;                                                                    \
    const int e = 2 * r + 1;                                                         \
    const int zlo = dim == 3 ? -r : 0, zhi = dim == 3 ? r : 0;                      \
    for (int dz = zlo; dz <= zhi; ++dz)                                              \
      for (int dy = -r; dy <= r; ++dy)                                               \
        for (int dx = -r; dx <= r; ++dx) {                                           \
          const int axes = (dz != 0) + (dy != 0) + (dx != 0);                        \
          if (kind == ORC_STAR && axes > 1) continue;                                \
          const size_t wi = ((size_t)(dz + (dim == 3 ? r : 0)) * e + (dy + r)) * e + \
                            (dx + r);                                                \
          const T wt = (T)w[wi];                                                     \
          const size_t at = c + (ptrdiff_t)dz * (ptrdiff_t)sz_ +                     \
                            (ptrdiff_t)dy * (ptrdiff_t)sy + dx;                      \
          acc = FMA(wt, in[at], acc);                                                \
        }                                                                            \
    return acc;                                                                      \
  }                                                                                  \
  void orc_step_##SUFFIX(const T* in, T* out, int sz, int r, const orc_stencil* st) { \
    const int p = sz + 2 * r;                                                        \
    const size_t sy = (size_t)p, splane = (size_t)p * p;                             \
    const int zlo = st->dim == 3 ? r : 0, zhi = st->dim == 3 ? r + sz : 1;           \
    for (int z = zlo; z < zhi; ++z)                                                  \
      for (int y = r; y < r + sz; ++y)                                               \
        for (int x = r; x < r + sz; ++x) {                                           \
          const size_t c = (size_t)z * splane + (size_t)y * sy + (size_t)x;          \
          out[c] = orc_point_##SUFFIX(in, c, sy, splane, r, st->dim, st->kind, st->w); \
        }                                                                            \
  }                                                                                  \
  void orc_run_##SUFFIX(const T* g, T* out, int sz, int r, const orc_stencil* st,    \
                        int steps) {                                                 \
    const int p = sz + 2 * r;                                                        \
    const size_t n = (size_t)p * p * (st->dim == 3 ? (size_t)p : 1);                 \
    T* a = (T*)malloc(n * sizeof(T));                                                \
    T* b = (T*)malloc(n * sizeof(T));                                                \
    memcpy(a, g, n * sizeof(T));                                                     \
    memcpy(b, g, n * sizeof(T));                                                     \
    T* src = a;                                                                      \
    T* dst = b;                                                                      \
    for (int s = 0; s < steps; ++s) {                                                \
      orc_step_##SUFFIX(src, dst, sz, r, st);                                        \
      T* t = src;                                                                    \
      src = dst;                                                                     \
      dst = t;                                                                       \
    }                                                                                \
    memcpy(out, src, n * sizeof(T));                                                 \
    free(a);                                                                         \
    free(b);                                                                         \
  }

ORC_DEFINE_STEP(f32, float, fmaf)
ORC_DEFINE_STEP(f64, double, fma)

/* Same per-point rule on a rectangular padded block of nz x ny x nx cells
 * (nz = 1 for 2D) whose outer r cells in every stencil dimension are held
 * constant -- the light-cone checker for full-size runs: a cut-out of the
 * grid with a margin of r*steps around a window evolves that window exactly
 * as the whole grid does (per-point arithmetic depends only on the
 * (2r+1)^dim neighbourhood; the contamination from the held margin travels r
 * cells per step). */
#define ORC_DEFINE_BLOCK(SUFFIX, T)                                                  \
  void orc_run_block_##SUFFIX(const T* g, T* out, int nz, int ny, int nx, int r,     \
                              const orc_stencil* st, int steps, const int* wlo,      \
                              const int* whi) {                                      \
    const size_t n = (size_t)nz * ny * nx;                                           \
    const size_t sy = (size_t)nx, splane = (size_t)nx * ny;                          \
    T* a = (T*)malloc(n * sizeof(T));                                                \
    T* b = (T*)malloc(n * sizeof(T));                                                \
    memcpy(a, g, n * sizeof(T));                                                     \
    memcpy(b, g, n * sizeof(T));                                                     \
    T* src = a;                                                                      \
    T* dst = b;                                                                      \
    const int d3 = st->dim == 3;                                                     \
    const int ext[3] = {nz, ny, nx};                                                 \
    for (int s = 1; s <= steps; ++s) {                                               \
      /* only the cells the window still depends on: window +- r*(steps-s) */        \
      int lo[3], hi[3];                                                              \
      for (int k = 0; k < 3; ++k) {                                                  \
        lo[k] = r;                                                                   \
        hi[k] = ext[k] - r;                                                          \
        if (wlo && whi) {                                                            \
          const int gr = r * (steps - s);                                            \
          if (wlo[k] - gr > lo[k]) lo[k] = wlo[k] - gr;                              \
          if (whi[k] + gr < hi[k]) hi[k] = whi[k] + gr;                              \
        }                                                                            \
      }                                                                              \
      if (!d3) {                                                                     \
        lo[0] = 0;                                                                   \
        hi[0] = 1;                                                                   \
      }                                                                              \
      _Pragma("omp parallel for collapse(2) schedule(static)")                       \
      for (int z = lo[0]; z < hi[0]; ++z)                                            \
        for (int y = lo[1]; y < hi[1]; ++y)                                          \
          for (int x = lo[2]; x < hi[2]; ++x) {                                      \
            const size_t c = (size_t)z * splane + (size_t)y * sy + (size_t)x;        \
            dst[c] = orc_point_##SUFFIX(src, c, sy, splane, r, st->dim, st->kind, st->w); \
          }                                                                          \
      T* t = src;                                                                    \
      src = dst;                                                                     \
      dst = t;                                                                       \
    }                                                                                \
    memcpy(out, src, n * sizeof(T));                                                 \
    free(a);                                                                         \
    free(b);                                                                         \
  }

ORC_DEFINE_BLOCK(f32, float)
ORC_DEFINE_BLOCK(f64, double)

uint64_t orc_fnv1a(const void* data, size_t bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xCBF29CE484222325ULL;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ULL;
  }
  return h;
}

/*
 * so2dr_oracle.h -- CPU restatement of the SO2DR reference arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product library links or calls
 * this code: it is the checker that tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py compare the CUDA path against.
 *
 * Parity pinning: the 2D fp32 paths are cross-checked bit-for-bit against the
 * reference itself (oracle/_ref/libso2dr_ref.so, compiled from
 * /root/reference/proj/src by oracle/Makefile) and against the golden
 * vectors in tests/golden/. 3D and fp64 have no reference implementation;
 * they are a restatement of the same per-point rules in (dz, dy, dx)
 * canonical order and are pinned only through the degenerate cases
 * (dz != 0 weights zero -> every z-plane equals the 2D reference; fp64
 * known-answer tests with exactly representable values).
 */
#ifndef SO2DR_ORACLE_H
#define SO2DR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* stencil kinds, same numbering as include/so2dr_cuda.h */
enum { ORC_BOX = 0, ORC_GRADIENT = 1, ORC_STAR = 2 };

/* Stencil description: `w` holds (2r+1)^dim weights in canonical order
 * (dz, dy, dx ascending; dx fastest). For ORC_STAR only the on-axis entries
 * are read. ORC_GRADIENT ignores w (pinned expression). */
typedef struct {
  int kind;
  int dim;    /* 2 or 3 */
  int radius; /* r */
  const double* w;
} orc_stencil;

/* proj/src/stencil.cpp:91-118 -- splitmix64 counter-based cell value. */
float orc_cell_value(uint64_t seed, int y, int x);
/* 3D extension: plane z uses seed ^ (z * golden), so plane 0 == 2D grid. */
float orc_cell_value3(uint64_t seed, int z, int y, int x);

/* Fill a padded grid (edge p = sz + 2r; p^dim cells, row-major) */
void orc_init_f32(float* g, int dim, int sz, int r, uint64_t seed);
void orc_init_f64(double* g, int dim, int sz, int r, uint64_t seed);

/* init values of a box of the padded grid (dim 2: z0 ignored, nz = 1) */
void orc_init_block_f32(float* g, int dim, int z0, int y0, int x0, int nz, int ny, int nx, uint64_t seed);
void orc_init_block_f64(double* g, int dim, int z0, int y0, int x0, int nz, int ny, int nx, uint64_t seed);

/* proj/src/stencil.cpp:146-160 (apply_step) generalised: one step over the
 * full interior, reading `in`, writing `out` (ring cells of out untouched). */
void orc_step_f32(const float* in, float* out, int sz, int r, const orc_stencil* st);
void orc_step_f64(const double* in, double* out, int sz, int r, const orc_stencil* st);

/* proj/src/stencil.cpp:162-174 (run_reference): `steps` ping-pong steps,
 * result written to `out` (may alias `g`). */
void orc_run_f32(const float* g, float* out, int sz, int r, const orc_stencil* st, int steps);
void orc_run_f64(const double* g, double* out, int sz, int r, const orc_stencil* st, int steps);

/* run_reference on a rectangular padded block (nz = 1 for dim 2): the outer
 * r cells of every stencil dimension are held constant. Used to check
 * windows of full-size runs (light-cone property, see so2dr_oracle.c). */
void orc_run_block_f32(const float* g, float* out, int nz, int ny, int nx, int r,
                       const orc_stencil* st, int steps, const int* wlo, const int* whi);
void orc_run_block_f64(const double* g, double* out, int nz, int ny, int nx, int r,
                       const orc_stencil* st, int steps, const int* wlo, const int* whi);
/* (wlo/whi: optional [z,y,x] window in block coordinates (z = 0..1 for 2D);
 * when given, step s only updates the window grown by r*(steps-s) -- the
 * cells the window still depends on; other cells of `out` are stale.) */

/* proj/src/stencil.cpp:176-186 -- FNV-1a 64 over raw bytes. */
uint64_t orc_fnv1a(const void* data, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif

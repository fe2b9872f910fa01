// k1_launch.h -- host-side launch interface of the K1 stencil kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Force-inline device lambdas: a lambda ptxas leaves out of line becomes a
// CALL whose ABI spills the whole pipeline state to local memory (seen on the
// fp64 star kernels: 1.5 KB stack frame, 25x slower).
#define SO2DR_INLINE __attribute__((always_inline))

namespace so2dr_dev {

// stencil kinds as the kernels see them (a box with zero off-axis weights is
// dispatched as KSTAR)
enum : int { KBOX = 0, KGRAD = 1, KSTAR = 2 };

// One fused k-step launch over a device field (see k1_2d.cuh / k1_3d.cuh for
// the semantics). For dim 3 "rows" are z-planes of plane_rows x cols cells
// (plane stride = plane_rows * pitch), and the y/x interior + region are the
// full plane interior (the engine only splits along z).
struct K1Launch {
  int dim = 2;
  int dtype = 0;  // 0 f32, 1 f64
  int kind = 0;   // KBOX/KGRAD/KSTAR
  int radius = 1;
  int steps = 1;
  const void* in = nullptr;
  void* out = nullptr;
  int64_t pitch = 0;  // elements per storage row
  int base = 0, rows = 0, cols = 0;
  int plane_rows = 0;  // 3D: rows per plane (padded edge)
  int y0 = 0, y1 = 0, x0 = 0, x1 = 0;
  int iy0 = 0, iy1 = 0, ix0 = 0, ix1 = 0;
  const double* w = nullptr;  // (2R+1)^dim weights, canonical order
};

// Largest step count one launch fuses for (dim, dtype, kind, radius); longer
// calls are split by the caller.
int k1_max_steps(int dim, int dtype, int kind, int radius);

// Launches K1. Returns cudaErrorInvalidValue for unsupported shapes.
cudaError_t k1_launch(const K1Launch& L, cudaStream_t stream);

// Algorithmic HBM bytes of one launch: every input row read once plus every
// output row written once (full padded width).
uint64_t k1_alg_bytes(const K1Launch& L);

cudaError_t launch_k1_2d_f32(const K1Launch& L, cudaStream_t stream);
cudaError_t launch_k1_2d_f64(const K1Launch& L, cudaStream_t stream);
cudaError_t launch_k1_3d_f32(const K1Launch& L, cudaStream_t stream);
cudaError_t launch_k1_3d_f64(const K1Launch& L, cudaStream_t stream);

int device_sm_count();

// Zeroed work counter for one persistent K1 launch on `stream`.
unsigned* k1_next_counter(cudaStream_t stream);

}  // namespace so2dr_dev

// 2D K1 dispatch by radius (instantiations live in k1_2d_{f32,f64}_r*.cu).
#include "k1_launch.h"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f32_r1(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r2(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r3(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f32_r4(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r1(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r2(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r3(const K1Launch& L, cudaStream_t s);
cudaError_t launch_k1_2d_f64_r4(const K1Launch& L, cudaStream_t s);

cudaError_t launch_k1_2d_f32(const K1Launch& L, cudaStream_t s) {
  switch (L.radius) {
    case 1: return launch_k1_2d_f32_r1(L, s);
    case 2: return launch_k1_2d_f32_r2(L, s);
    case 3: return launch_k1_2d_f32_r3(L, s);
    case 4: return launch_k1_2d_f32_r4(L, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_k1_2d_f64(const K1Launch& L, cudaStream_t s) {
  switch (L.radius) {
    case 1: return launch_k1_2d_f64_r1(L, s);
    case 2: return launch_k1_2d_f64_r2(L, s);
    case 3: return launch_k1_2d_f64_r3(L, s);
    case 4: return launch_k1_2d_f64_r4(L, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace so2dr_dev

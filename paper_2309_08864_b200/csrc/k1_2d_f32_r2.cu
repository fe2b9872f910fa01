// 2D K1 instantiations: float, radius 2.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f32_r2(const K1Launch& L, cudaStream_t s) { return launch_2d_r<float, 2>(L, s); }
}  // namespace so2dr_dev

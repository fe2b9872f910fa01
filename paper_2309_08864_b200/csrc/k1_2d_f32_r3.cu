// 2D K1 instantiations: float, radius 3.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f32_r3(const K1Launch& L, cudaStream_t s) { return launch_2d_r<float, 3>(L, s); }
}  // namespace so2dr_dev

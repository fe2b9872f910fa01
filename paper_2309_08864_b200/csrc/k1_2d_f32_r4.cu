// 2D K1 instantiations: float, radius 4.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f32_r4(const K1Launch& L, cudaStream_t s) { return launch_2d_r<float, 4>(L, s); }
}  // namespace so2dr_dev

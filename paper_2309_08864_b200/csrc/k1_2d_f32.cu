// 2D K1 instantiations, fp32.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f32(const K1Launch& L, cudaStream_t stream) { return launch_2d<float>(L, stream); }
}  // namespace so2dr_dev

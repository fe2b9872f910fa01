// 2D K1 instantiations: double, radius 1.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f64_r1(const K1Launch& L, cudaStream_t s) { return launch_2d_r<double, 1>(L, s); }
}  // namespace so2dr_dev

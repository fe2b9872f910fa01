// 2D K1 instantiations, fp64.
#include "k1_2d_impl.cuh"
namespace so2dr_dev {
cudaError_t launch_k1_2d_f64(const K1Launch& L, cudaStream_t stream) { return launch_2d<double>(L, stream); }
}  // namespace so2dr_dev

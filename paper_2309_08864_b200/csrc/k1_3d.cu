// 3D K1 kernels -- placeholder until the z-streamed kernel lands.
#include "k1_launch.h"
namespace so2dr_dev {
cudaError_t launch_k1_3d_f32(const K1Launch&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_k1_3d_f64(const K1Launch&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace so2dr_dev

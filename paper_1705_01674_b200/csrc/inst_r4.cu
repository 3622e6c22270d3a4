// Instantiation of the pass kernels for radius r = 4 (see sgwls_pass.cuh).
#include "sgwls_pass.cuh"

namespace sgwls_b200 {
template cudaError_t launch_pass_r<4>(const PassLaunch& pl, cudaStream_t st);
}  // namespace sgwls_b200

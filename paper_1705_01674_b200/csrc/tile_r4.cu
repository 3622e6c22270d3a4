// Instantiation of the CTA-tiled fast path for radius r = 4 (see sgwls_tile.cuh).
#include "sgwls_tile.cuh"

namespace sgwls_b200 {
namespace tile {
template cudaError_t launch_tile_r<4>(const PassLaunch& pl, cudaStream_t st);
}  // namespace tile
}  // namespace sgwls_b200

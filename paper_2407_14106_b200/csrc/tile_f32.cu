// float instantiation of the tile-scheduled sparse attention kernels.
#include "tile_launch.cuh"

namespace gte_b200 {

cudaError_t launch_tile_f32(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st, int* launches) {
  return launch_tile_t<float>(which, a, lph, lpn, st, launches);
}

}  // namespace gte_b200

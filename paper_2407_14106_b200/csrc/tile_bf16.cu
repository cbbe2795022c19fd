// __nv_bfloat16 instantiation of the tile-scheduled sparse attention kernels.
#include "tile_launch.cuh"

namespace gte_b200 {

cudaError_t launch_tile_bf16(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st, int* launches) {
  return launch_tile_t<__nv_bfloat16>(which, a, lph, lpn, st, launches);
}

}  // namespace gte_b200

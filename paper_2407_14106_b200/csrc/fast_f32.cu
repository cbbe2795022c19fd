// float instantiation of the memory-level-parallel sparse attention kernels.
#include "fast_launch.cuh"

namespace gte_b200 {

cudaError_t launch_fast_f32(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st) {
  return launch_fast_t<float>(which, a, lph, lpn, st);
}

}  // namespace gte_b200

// __nv_bfloat16 instantiation of the memory-level-parallel sparse attention kernels.
#include "fast_launch.cuh"

namespace gte_b200 {

cudaError_t launch_fast_bf16(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st) {
  return launch_fast_t<__nv_bfloat16>(which, a, lph, lpn, st);
}

}  // namespace gte_b200

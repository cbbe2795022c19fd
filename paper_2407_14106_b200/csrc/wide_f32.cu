// float instantiation of the padded tile kernels (attn_wide.cuh).
#include "wide_launch.cuh"

namespace gte_b200 {

cudaError_t launch_wide_f32(int which, const SparseArgs& a, int head_bytes, int piece_bytes, int lpn, cudaStream_t st,
                           int* launches) {
  return launch_wide_t<float>(which, a, head_bytes, piece_bytes, lpn, st, launches);
}

}  // namespace gte_b200

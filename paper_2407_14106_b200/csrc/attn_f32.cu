// float instantiation of the sparse graph-attention kernels (see attn_sparse.cuh).
#include "attn_launch.cuh"

namespace gte_b200 {

cudaError_t launch_sparse_f32(int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st) {
  return launch_sparse_t<float>(which, a, dht, lpn, st);
}

}  // namespace gte_b200

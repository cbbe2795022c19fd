// Row-gather throughput ceiling on B200 for the sparse kernels' access
// pattern: per edge, 8 lanes each load one 16-byte piece of a 128-byte K row
// and of a 128-byte V row (bf16, H*dh = 64), EPL = 4 edges per 8-lane slot
// per step, rows picked by an index array. No math beyond an XOR fold (kept
// live by one store per thread). Reports requested bytes / time, i.e. the
// same quantity as bench.py's l2_gather.achieved_gbs. f32 rows: 16 lanes x 16 B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC gather_bw.cu -o libgather_bw.so
#include <cuda_runtime.h>
#include <stdint.h>

template <int EPL, int PR>  // PR: 16-byte pieces per row (8: bf16 x 64, 16: f32 x 64)
__global__ void __launch_bounds__(256) gather_kernel(const uint4* __restrict__ K, const uint4* __restrict__ V,
                                                     const int* __restrict__ idx, int64_t E, uint4* sink) {
  constexpr int kShift = PR == 8 ? 3 : 4;
  const int lane = threadIdx.x & 31, piece = lane & (PR - 1);
  const int64_t slot = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> kShift;
  const int64_t nslots = ((int64_t)gridDim.x * blockDim.x) >> kShift;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t e0 = slot * EPL; e0 < E; e0 += nslots * EPL) {
    uint4 k[EPL], v[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int64_t e = e0 + u < E ? e0 + u : E - 1;
      const uint32_t j = (uint32_t)__ldg(idx + e);
      k[u] = __ldg(K + (size_t)j * PR + piece);
      v[u] = __ldg(V + (size_t)j * PR + piece);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      acc.x ^= k[u].x ^ v[u].y;
      acc.y ^= k[u].y ^ v[u].z;
      acc.z ^= k[u].z ^ v[u].w;
      acc.w ^= k[u].w ^ v[u].x;
    }
  }
  if ((acc.x & 0xfffffff) == 0x1234567) sink[threadIdx.x] = acc;  // practically never; keeps the loads live
}

extern "C" int gather_bw(const void* K, const void* V, const int* idx, int64_t E, void* sink, int blocks,
                         int reps, float* ms, int row_bytes) {
  auto go = [&] {
    if (row_bytes == 256)
      gather_kernel<4, 16><<<blocks, 256>>>((const uint4*)K, (const uint4*)V, idx, E, (uint4*)sink);
    else
      gather_kernel<4, 8><<<blocks, 256>>>((const uint4*)K, (const uint4*)V, idx, E, (uint4*)sink);
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  go();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) go();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  *ms /= reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (int)cudaGetLastError();
}

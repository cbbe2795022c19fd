// Trainer glue around the attention kernels: the pattern's
// pad loops and SPD bias buckets (proj/src/model.cpp:76-83, 407-423,
// 447-463; SpdTable::lookup graph.cpp:208-214), the bias gather from the
// per-layer bucket table (model.cpp:520-523) and the table gradient.
//
//   gte_pattern_buckets    one thread per attended pair: (r, c) execution
//                          coordinates -> original ids through perm.inverse,
//                          0 self / 1 global token / unreachable for pads /
//                          binary search in the SPD row (absent: unreachable)
//   gte_bias_from_table    bias[e] = table[bucket[e]]
//   gte_dbias_to_table     dtable[b] = sum of dbias[e] over bucket[e] == b:
//                          per-CTA partials in shared memory, then one
//                          fixed-order pass (deterministic, no float atomics)
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define GLCUDA(expr)                                                                                  \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                 \
  } while (0)

namespace {

constexpr int kMaxBuckets = 64;
constexpr int kTableGrid = 296;

__device__ __forceinline__ int32_t row_of_edge(const int32_t* __restrict__ rp, int32_t rows, int32_t e) {
  int32_t lo = 0, hi = rows;  // last r with rp[r] <= e
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (__ldg(rp + mid) <= e) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void buckets_kernel(int32_t rows, int32_t nnz, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ cols, const int64_t* __restrict__ inv, int64_t global,
                               int64_t spd_n, const int64_t* __restrict__ sro, const int64_t* __restrict__ scol,
                               const uint16_t* __restrict__ sdist, int32_t unreachable, int32_t* __restrict__ out) {
  for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x) {
    const int32_t r = row_of_edge(rp, rows, e);
    const int64_t i = __ldg(inv + r), j = __ldg(inv + __ldg(cols + e));
    int32_t b;
    if (i == j) {
      b = 0;
    } else if (i == global || j == global) {
      b = 1;
    } else if (i >= spd_n || j >= spd_n) {
      b = unreachable;
    } else {
      int64_t lo = __ldg(sro + i), hi = __ldg(sro + i + 1);
      const int64_t end = hi;
      while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(scol + mid) < j) lo = mid + 1; else hi = mid;
      }
      b = (lo < end && __ldg(scol + lo) == j) ? (int32_t)__ldg(sdist + lo) : unreachable;
    }
    out[e] = b;
  }
}

__global__ void bias_gather_kernel(int32_t nnz, const int32_t* __restrict__ bucket, const float* __restrict__ table,
                                   int32_t nb, float* __restrict__ bias) {
  __shared__ float t[kMaxBuckets];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) t[i] = table[i];
  __syncthreads();
  for (int32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x)
    bias[e] = t[__ldg(bucket + e)];
}

// pass 1: CTA c sums its contiguous edge range per bucket (warp partials in a
// fixed order) -> part[c][b]; pass 2: out[b] = sum_c part[c][b] in c order
__global__ void table_partial_kernel(int32_t nnz, const int32_t* __restrict__ bucket, const float* __restrict__ dbias,
                                     int32_t nb, float* __restrict__ part) {
  __shared__ float acc[8][kMaxBuckets];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * kMaxBuckets; i += blockDim.x) acc[i / kMaxBuckets][i % kMaxBuckets] = 0.f;
  __syncthreads();
  const int64_t per = ((int64_t)nnz + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = e0 + per < nnz ? e0 + per : nnz;
  // each warp owns a strided set of 32-edge chunks; lanes reduce per bucket
  for (int64_t base = e0 + (int64_t)warp * 32; base < e1; base += 8 * 32) {
    const int64_t e = base + lane;
    const int b = e < e1 ? __ldg(bucket + e) : -1;
    const float v = e < e1 ? __ldg(dbias + e) : 0.f;
    // lane 0 adds the chunk's values bucket by bucket in lane order
    for (int l = 0; l < 32; ++l) {
      const int bl = __shfl_sync(0xffffffffu, b, l);
      const float vl = __shfl_sync(0xffffffffu, v, l);
      if (lane == 0 && bl >= 0) acc[warp][bl] += vl;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += acc[w][b];
    part[(int64_t)blockIdx.x * nb + b] = s;
  }
}

__global__ void table_final_kernel(int32_t parts, int32_t nb, const float* __restrict__ part, float* __restrict__ out) {
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < parts; ++c) s += part[(int64_t)c * nb + b];
    out[b] = s;
  }
}

}  // namespace

extern "C" {

int gte_extend_with_pad_loops_host(int64_t rows, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                                   int64_t s_pad, int64_t* out_row_off, int64_t* out_cols) {
  // model.cpp:76-83: rows [rows, s_pad) get a single self-loop each.
  // out_row_off [max(rows, s_pad) + 1], out_cols [nnz + max(0, s_pad - rows)]
  if (rows < 0 || nnz < 0) return set_error(GTE_CONFIG, "extend_with_pad_loops: negative size");
  for (int64_t r = 0; r <= rows; ++r) out_row_off[r] = row_off[r];
  for (int64_t e = 0; e < nnz; ++e) out_cols[e] = cols[e];
  for (int64_t r = rows; r < s_pad; ++r) {
    out_cols[out_row_off[r]] = r;
    out_row_off[r + 1] = out_row_off[r] + 1;
  }
  return GTE_OK;
}

int gte_pattern_buckets(gte_ctx* ctx, int64_t rows, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                        const int64_t* d_perm_inverse, int64_t global_index, int64_t spd_n,
                        const int64_t* d_spd_row_off, const int64_t* d_spd_cols, const uint16_t* d_spd_dist,
                        int64_t max_dist, int32_t* d_buckets) {
  if (rows < 0 || nnz < 0 || rows >= INT32_MAX || nnz >= INT32_MAX)
    return set_error(GTE_CONFIG, "pattern_buckets: bad pattern size");
  if (max_dist < 0 || max_dist + 2 > kMaxBuckets) return set_error(GTE_CONFIG, "pattern_buckets: max_dist out of range");
  if (nnz == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const int64_t g = (nnz + 255) / 256;
  buckets_kernel<<<(unsigned)(g < 148 * 64 ? g : 148 * 64), 256, 0, st>>>(
      (int32_t)rows, (int32_t)nnz, d_row_ptr, d_cols, d_perm_inverse, global_index, spd_n, d_spd_row_off,
      d_spd_cols, d_spd_dist, (int32_t)(max_dist + 1), d_buckets);
  ctx_launch_counter(ctx) += 1;
  GLCUDA(cudaGetLastError());
  return GTE_OK;
}

int gte_bias_from_table(gte_ctx* ctx, int64_t nnz, const int32_t* d_buckets, const float* d_table, int64_t n_buckets,
                        float* d_bias) {
  if (n_buckets < 1 || n_buckets > kMaxBuckets) return set_error(GTE_CONFIG, "bias_from_table: bucket count out of range");
  if (nnz >= INT32_MAX) return set_error(GTE_CONFIG, "bias_from_table: pattern too large");
  if (nnz <= 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const int64_t g = (nnz + 255) / 256;
  bias_gather_kernel<<<(unsigned)(g < 148 * 16 ? g : 148 * 16), 256, 0, st>>>((int32_t)nnz, d_buckets, d_table,
                                                                             (int32_t)n_buckets, d_bias);
  ctx_launch_counter(ctx) += 1;
  GLCUDA(cudaGetLastError());
  return GTE_OK;
}

int gte_dbias_to_table(gte_ctx* ctx, int64_t nnz, const int32_t* d_buckets, const float* d_dbias, int64_t n_buckets,
                       float* d_table_grad, float* d_workspace /* [296 * n_buckets] */) {
  if (n_buckets < 1 || n_buckets > kMaxBuckets) return set_error(GTE_CONFIG, "dbias_to_table: bucket count out of range");
  if (nnz >= INT32_MAX) return set_error(GTE_CONFIG, "dbias_to_table: pattern too large");
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  table_partial_kernel<<<kTableGrid, 256, 0, st>>>((int32_t)(nnz > 0 ? nnz : 0), d_buckets, d_dbias,
                                                   (int32_t)n_buckets, d_workspace);
  table_final_kernel<<<1, 64, 0, st>>>(kTableGrid, (int32_t)n_buckets, d_workspace, d_table_grad);
  ctx_launch_counter(ctx) += 2;
  GLCUDA(cudaGetLastError());
  return GTE_OK;
}

}  // extern "C"

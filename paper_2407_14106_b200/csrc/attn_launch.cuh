// Compile-time dispatch for the sparse attention kernels. Each dtype is
// instantiated in its own translation unit (attn_f32.cu, attn_bf16.cu,
// attn_f64.cu) so nvcc builds them in parallel.
#pragma once

#include <cstdlib>

#include "attn_sparse.cuh"

namespace gte_b200 {

enum SparseKernel { kFwd = 0, kBwdRows = 1, kBwdCols = 2 };

// Rows (resp. columns) per CTA: a contiguous range per CTA so a cluster-ordered
// sequence's gathers stay L1-resident; GTE_ROWS_PER_CTA overrides (tuning).
inline int64_t rows_per_cta_for(int64_t S) {
  static const int64_t env = [] {
    const char* e = getenv("GTE_ROWS_PER_CTA");
    return e ? atoll(e) : 0LL;
  }();
  int64_t r = env > 0 ? env : 128;
  // keep at least ~4 CTAs per SM for balance on short sequences
  while (r > 8 && (S + r - 1) / r < 148 * 4) r >>= 1;
  return r < 8 ? 8 : r;
}

template <typename T, int DHT, int LPN>
cudaError_t launch_one(int which, const SparseArgs& a, cudaStream_t st) {
  constexpr int kBlock = 256;
  SparseArgs b = a;
  b.rows_per_cta = rows_per_cta_for(a.S);
  int64_t grid = (a.S + b.rows_per_cta - 1) / b.rows_per_cta;
  if (grid > (1LL << 30)) grid = 1LL << 30;
  if (grid < 1) grid = 1;
  switch (which) {
    case kFwd: sparse_fwd_kernel<T, DHT, LPN><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
    case kBwdRows: sparse_bwd_rows_kernel<T, DHT, LPN><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
    default: sparse_bwd_cols_kernel<T, DHT, LPN><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
  }
  return cudaGetLastError();
}

template <typename T, int DHT>
cudaError_t launch_lpn(int which, const SparseArgs& a, int lpn, cudaStream_t st) {
  switch (lpn) {
    case 1: return launch_one<T, DHT, 1>(which, a, st);
    case 2: return launch_one<T, DHT, 2>(which, a, st);
    case 4: return launch_one<T, DHT, 4>(which, a, st);
    case 8: return launch_one<T, DHT, 8>(which, a, st);
    case 16: return launch_one<T, DHT, 16>(which, a, st);
    case 32: return launch_one<T, DHT, 32>(which, a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
cudaError_t launch_sparse_t(int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st) {
  switch (dht) {
    case 8: return launch_lpn<T, 8>(which, a, lpn, st);
    case 16: return launch_lpn<T, 16>(which, a, lpn, st);
    case 32: return launch_lpn<T, 32>(which, a, lpn, st);
    case 64: return launch_lpn<T, 64>(which, a, lpn, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sparse_f32(int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st);
cudaError_t launch_sparse_bf16(int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st);
cudaError_t launch_sparse_f64(int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st);
cudaError_t launch_finite_rows(int dtype, const void* k, const void* v, const int32_t* rows, int nrows,
                               int64_t ldq, int64_t ldv, int64_t wq, int64_t wv, int* err, cudaStream_t st);

}  // namespace gte_b200

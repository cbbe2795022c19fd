// Dispatch for the memory-level-parallel kernels (attn_fast.cuh).
#pragma once

#include "attn_rowslot.cuh"
#include "attn_launch.cuh"

namespace gte_b200 {

#ifndef GTE_FAST_EPL
#define GTE_FAST_EPL 8
#endif
#ifndef GTE_SLOT_EPL
#define GTE_SLOT_EPL 4
#endif

template <typename T, int LPH, int LPN>
cudaError_t launch_fast_one(int which, const SparseArgs& a, cudaStream_t st) {
  constexpr int kBlock = 256;
  // a chunk (SLOTS * EPL edges) must fit the 32 column indices a warp loads
  constexpr int EPL = GTE_FAST_EPL < LPN ? GTE_FAST_EPL : LPN;
  SparseArgs b = a;
  b.rows_per_cta = rows_per_cta_for(a.S);
  int64_t grid = (a.S + b.rows_per_cta - 1) / b.rows_per_cta;
  if (grid > (1LL << 30)) grid = 1LL << 30;
  if (grid < 1) grid = 1;
  static const bool warp_rows = [] {
    const char* e = getenv("GTE_SCHED");
    return e && e[0] == 'w';
  }();
  static const int slot_epl = [] {
    const char* e = getenv("GTE_SLOT_EPL");
    return e ? atoi(e) : GTE_SLOT_EPL;
  }();
  if (!warp_rows) {  // default: row-slot schedule (attn_rowslot.cuh)
    if (slot_epl >= 8) {
      switch (which) {
        case kFwd: slot_fwd_kernel<T, LPH, LPN, 8><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
        case kBwdRows: slot_bwd_rows_kernel<T, LPH, LPN, 8><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
        default: slot_bwd_cols_kernel<T, LPH, LPN, 8><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
      }
      return cudaGetLastError();
    }
    switch (which) {
      case kFwd: slot_fwd_kernel<T, LPH, LPN, 4><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
      case kBwdRows: slot_bwd_rows_kernel<T, LPH, LPN, 4><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
      default: slot_bwd_cols_kernel<T, LPH, LPN, 4><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
    }
    return cudaGetLastError();
  }
  switch (which) {
    case kFwd: fast_fwd_kernel<T, LPH, LPN, EPL><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
    case kBwdRows: fast_bwd_rows_kernel<T, LPH, LPN, EPL><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
    default: fast_bwd_cols_kernel<T, LPH, LPN, EPL><<<(unsigned)grid, kBlock, 0, st>>>(b); break;
  }
  return cudaGetLastError();
}

template <typename T, int LPH>
cudaError_t launch_fast_lpn(int which, const SparseArgs& a, int lpn, cudaStream_t st) {
  switch (lpn) {
    case 1: if constexpr (LPH <= 1) return launch_fast_one<T, LPH, 1>(which, a, st); break;
    case 2: if constexpr (LPH <= 2) return launch_fast_one<T, LPH, 2>(which, a, st); break;
    case 4: if constexpr (LPH <= 4) return launch_fast_one<T, LPH, 4>(which, a, st); break;
    case 8: if constexpr (LPH <= 8) return launch_fast_one<T, LPH, 8>(which, a, st); break;
    case 16: return launch_fast_one<T, LPH, 16>(which, a, st);
    case 32: return launch_fast_one<T, LPH, 32>(which, a, st);
    default: break;
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_fast_t(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st) {
  switch (lph) {
    case 1: return launch_fast_lpn<T, 1>(which, a, lpn, st);
    case 2: return launch_fast_lpn<T, 2>(which, a, lpn, st);
    case 4: return launch_fast_lpn<T, 4>(which, a, lpn, st);
    case 8: return launch_fast_lpn<T, 8>(which, a, lpn, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fast_f32(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st);
cudaError_t launch_fast_bf16(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st);

}  // namespace gte_b200

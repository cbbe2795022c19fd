// Dispatch for the padded tile kernels (attn_wide.cuh): one tile launch per
// pass (grid = tiles of the execution plan) plus, when the plan has hub rows
// (columns), the hub kernels of attn_tile.cuh with the matching 16-byte
// geometry. PB = bytes per lane piece (16: LDG.128, 32: LDG.256).
#pragma once

#include "attn_wide.cuh"
#include "tile_launch.cuh"

namespace gte_b200 {

template <int PB> struct WideCfg {
  static constexpr int kEplFwd = 4, kEplRows = 4, kEplCols = PB == 16 ? 4 : 2;
#ifndef GTE_WIDE_MINB
#define GTE_WIDE_MINB 4
#endif
  static constexpr int kMinBlocks = PB == 16 ? GTE_WIDE_MINB : 2;  // 64 / 128 registers per thread
  static constexpr int kMinBlocksCols = PB == 16 ? 3 : 2;
};

template <typename T, int PB, int HPP, int LPH, int LPN, bool WM>
cudaError_t launch_wide_one(int which, const SparseArgs& a, cudaStream_t st, int* launches) {
  using C = WideCfg<PB>;
  constexpr int MB = C::kMinBlocks;
  const size_t smem = wide_smem_bytes();
  cudaError_t e = cudaSuccess;
  const int nt = which == kBwdCols ? a.n_tiles_c : a.n_tiles;
  const int nh = which == kBwdCols ? a.n_hubs_c : a.n_hubs;
  if (nt > 0) {
    switch (which) {
      case kFwd: e = tile_go(wide_fwd_kernel<T, PB, HPP, LPH, LPN, C::kEplFwd, WM, MB>, nt, smem, a, st); break;
      case kBwdRows:
        e = tile_go(wide_bwd_rows_kernel<T, PB, HPP, LPH, LPN, C::kEplRows, WM, MB>, nt, smem, a, st);
        break;
      default: e = tile_go(wide_bwd_cols_kernel<T, PB, HPP, LPH, LPN, C::kEplCols, WM, C::kMinBlocksCols>, nt, smem, a, st); break;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  if (nh > 0) {
    // hub kernels: 16-byte pieces, LPH16 lanes per head, LPN16 lanes per row
    constexpr int kHeadBytes = (PB / HPP) * LPH;
    constexpr int LPH16 = kHeadBytes / 16;
    constexpr int LPN16 = LPN * PB / 16;
    if constexpr (LPN16 <= 32 && LPH16 >= 1) {
      switch (which) {
        case kFwd: hub_fwd_kernel<T, LPH16, LPN16, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
        case kBwdRows: hub_bwd_rows_kernel<T, LPH16, LPN16, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
        default: hub_bwd_cols_kernel<T, LPH16, LPN16, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
      }
      e = cudaGetLastError();
      ++*launches;
    } else {
      e = cudaErrorInvalidValue;
    }
  }
  return e;
}

template <typename T, int PB, int HPP, int LPH>
cudaError_t launch_wide_lpn(int which, const SparseArgs& a, int lpn, cudaStream_t st, int* launches) {
  switch (lpn) {
#define GTE_WIDE_CASE(L)                                                              \
  case L:                                                                             \
    if constexpr (L * PB / 16 <= 32 && L >= LPH)                                      \
      return a.wmult ? launch_wide_one<T, PB, HPP, LPH, L, true>(which, a, st, launches) \
                     : launch_wide_one<T, PB, HPP, LPH, L, false>(which, a, st, launches); \
    break;
    GTE_WIDE_CASE(4)
    GTE_WIDE_CASE(8)
    GTE_WIDE_CASE(16)
    GTE_WIDE_CASE(32)
#undef GTE_WIDE_CASE
    default: break;
  }
  return cudaErrorInvalidValue;
}

// head_bytes = dh * sizeof(T); piece bytes 16 or 32
template <typename T>
cudaError_t launch_wide_t(int which, const SparseArgs& a, int head_bytes, int piece_bytes, int lpn, cudaStream_t st,
                          int* launches) {
  if (piece_bytes == 16) {
    switch (head_bytes) {
      case 16: return launch_wide_lpn<T, 16, 1, 1>(which, a, lpn, st, launches);
      case 32: return launch_wide_lpn<T, 16, 1, 2>(which, a, lpn, st, launches);
      case 64: return launch_wide_lpn<T, 16, 1, 4>(which, a, lpn, st, launches);
      default: break;
    }
  } else {
    switch (head_bytes) {
      case 16: if constexpr (sizeof(T) == 2) return launch_wide_lpn<T, 32, 2, 1>(which, a, lpn, st, launches); break;
      case 32: return launch_wide_lpn<T, 32, 1, 1>(which, a, lpn, st, launches);
      case 64: return launch_wide_lpn<T, 32, 1, 2>(which, a, lpn, st, launches);
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_wide_f32(int which, const SparseArgs& a, int head_bytes, int piece_bytes, int lpn, cudaStream_t st,
                            int* launches);
cudaError_t launch_wide_bf16(int which, const SparseArgs& a, int head_bytes, int piece_bytes, int lpn,
                             cudaStream_t st, int* launches);

}  // namespace gte_b200

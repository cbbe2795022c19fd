// Dispatch for the tile-scheduled kernels (attn_tile.cuh): per pass one tile
// launch (grid = tiles of the execution plan) and one hub launch (grid = hub
// rows/columns), each only if non-empty. Returns the number of launches.
#pragma once

#include <utility>
#include <vector>

#include "attn_launch.cuh"
#include "attn_tile.cuh"

namespace gte_b200 {

template <typename K>
cudaError_t tile_go(K kernel, int grid, size_t smem, const SparseArgs& a, cudaStream_t st) {
  // dynamic smem above 48 KB needs an opt-in per kernel (per instantiation
  // and per size: the attribute is set once for the largest size asked)
  static thread_local std::vector<std::pair<const void*, size_t>> done;
  if (smem > 48 * 1024) {
    bool ok = false;
    for (auto& d : done)
      if (d.first == reinterpret_cast<const void*>(kernel) && d.second >= smem) ok = true;
    if (!ok) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      done.emplace_back(reinterpret_cast<const void*>(kernel), smem);
    }
  }
  kernel<<<(unsigned)grid, kTileThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int LPH, int LPN, int EPL, bool WM>
cudaError_t launch_tile_one(int which, const SparseArgs& a, cudaStream_t st, int* launches) {
  cudaError_t e = cudaSuccess;
  const int nt = which == kBwdCols ? a.n_tiles_c : a.n_tiles;
  const int nh = which == kBwdCols ? a.n_hubs_c : a.n_hubs;
  if (nt > 0) {
    const size_t smem = tile_smem_bytes();
    switch (which) {
      case kFwd: e = tile_go(tile_fwd_kernel<T, LPH, LPN, EPL, WM>, nt, smem, a, st); break;
      case kBwdRows: e = tile_go(tile_bwd_rows_kernel<T, LPH, LPN, EPL, WM>, nt, smem, a, st); break;
      default: e = tile_go(tile_bwd_cols_kernel<T, LPH, LPN, EPL, WM>, nt, smem, a, st); break;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  if (nh > 0) {
    switch (which) {
      case kFwd: hub_fwd_kernel<T, LPH, LPN, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
      case kBwdRows: hub_bwd_rows_kernel<T, LPH, LPN, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
      default: hub_bwd_cols_kernel<T, LPH, LPN, 4, WM><<<nh, kTileThreads, 0, st>>>(a); break;
    }
    e = cudaGetLastError();
    ++*launches;
  }
  return e;
}

template <typename T, int LPH, int LPN>
cudaError_t launch_tile_wm(int which, const SparseArgs& a, cudaStream_t st, int* launches) {
  return a.wmult ? launch_tile_one<T, LPH, LPN, kTileEpl, true>(which, a, st, launches)
                 : launch_tile_one<T, LPH, LPN, kTileEpl, false>(which, a, st, launches);
}

template <typename T, int LPH>
cudaError_t launch_tile_lpn(int which, const SparseArgs& a, int lpn, cudaStream_t st, int* launches) {
  switch (lpn) {
    case 1: if constexpr (LPH <= 1) return launch_tile_wm<T, LPH, 1>(which, a, st, launches); break;
    case 2: if constexpr (LPH <= 2) return launch_tile_wm<T, LPH, 2>(which, a, st, launches); break;
    case 4: if constexpr (LPH <= 4) return launch_tile_wm<T, LPH, 4>(which, a, st, launches); break;
    case 8: if constexpr (LPH <= 8) return launch_tile_wm<T, LPH, 8>(which, a, st, launches); break;
    case 16: return launch_tile_wm<T, LPH, 16>(which, a, st, launches);
    case 32: return launch_tile_wm<T, LPH, 32>(which, a, st, launches);
    default: break;
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_tile_t(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st, int* launches) {
  switch (lph) {
    case 1: return launch_tile_lpn<T, 1>(which, a, lpn, st, launches);
    case 2: return launch_tile_lpn<T, 2>(which, a, lpn, st, launches);
    case 4: return launch_tile_lpn<T, 4>(which, a, lpn, st, launches);
    case 8: return launch_tile_lpn<T, 8>(which, a, lpn, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tile_f32(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st, int* launches);
cudaError_t launch_tile_bf16(int which, const SparseArgs& a, int lph, int lpn, cudaStream_t st, int* launches);

}  // namespace gte_b200

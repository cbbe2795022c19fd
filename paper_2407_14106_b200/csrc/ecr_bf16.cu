// Instantiation + launch of the ECR sub-block kernels (ecr_tile.cuh), bf16.
#include "ecr_tile.cuh"

namespace gte_b200 {

namespace {
template <int H, int DH, bool WM>
cudaError_t go(bool bwd, const EcrArgs& a, cudaStream_t st) {
  const size_t smem = ecr_smem_bytes<H, DH>(bwd);
  auto kf = ecr_fwd_kernel<H, DH, WM>;
  auto kb = ecr_bwd_kernel<H, DH, WM>;
  const void* fn = bwd ? reinterpret_cast<const void*>(kb) : reinterpret_cast<const void*>(kf);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)((a.n_blocks + kEcrWarps - 1) / kEcrWarps);
  if (bwd) kb<<<grid, kEcrWarps * 32, smem, st>>>(a);
  else kf<<<grid, kEcrWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}
template <int H, int DH>
cudaError_t go_wm(bool bwd, const EcrArgs& a, cudaStream_t st) {
  return a.wmult ? go<H, DH, true>(bwd, a, st) : go<H, DH, false>(bwd, a, st);
}
}  // namespace

bool ecr_eligible(int H, int dk, int dv) {
  return dk == dv && (dk == 8 || dk == 16) && (H * dk == 64 || H * dk == 128);
}

cudaError_t launch_ecr_bf16(bool bwd, const EcrArgs& a, cudaStream_t st) {
  if (a.n_blocks <= 0) return cudaSuccess;
  switch (a.H * 100 + a.dh) {
    case 808: return go_wm<8, 8>(bwd, a, st);
    case 416: return go_wm<4, 16>(bwd, a, st);
    case 1608: return go_wm<16, 8>(bwd, a, st);
    case 816: return go_wm<8, 16>(bwd, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gte_b200

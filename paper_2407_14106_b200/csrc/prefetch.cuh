// L2 warm-up for the gathered operands of a sparse-attention pass.
//
// ncu on the row-slot kernels: every step of a warp waits for the slowest of
// its ~32 row gathers, and ~15% of gathers go to DRAM, so each step pays a
// DRAM round trip. The gathered tensors (K, V for the forward / CSR pass; Q,
// dO for the CSC pass) are small next to the 126 MB L2 (64 MB at S = 256K,
// bf16), so a bulk prefetch issued first — one thread per CTA streaming
// `cp.async.bulk.prefetch.L2` (TMA) over its slice — turns nearly all gathers
// into L2 hits at the price of one sequential read of those tensors.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gte_b200 {

struct PrefetchArgs {
  const char* ptr[4];
  uint64_t bytes[4];
  int n;
};

__global__ void l2_prefetch_kernel(PrefetchArgs a) {
  if (threadIdx.x != 0) return;
  constexpr uint64_t kChunk = 64 * 1024;  // per bulk-prefetch instruction
  for (int t = 0; t < a.n; ++t) {
    const uint64_t total = a.bytes[t] & ~uint64_t(15);
    const uint64_t per = ((total / gridDim.x) + kChunk - 1) / kChunk * kChunk;
    const uint64_t b0 = (uint64_t)blockIdx.x * per;
    const uint64_t b1 = b0 + per < total ? b0 + per : total;
    for (uint64_t off = b0; off < b1; off += kChunk) {
      const uint64_t len = (b1 - off) < kChunk ? (b1 - off) : kChunk;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.ptr[t] + off), "r"((uint32_t)len) : "memory");
    }
  }
}

}  // namespace gte_b200

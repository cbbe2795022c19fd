// Throughput of the legacy warp-level tensor-core path on sm_100a:
// mma.sync m16n8k16 / m16n8k8 (bf16 -> f32) and movmatrix.trans, per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k16(float* out, int iters) {
  float d[4][4] = {};
  uint32_t a = threadIdx.x, b = threadIdx.x * 3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3]) : "r"(a), "r"(b));
  float s = 0; for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k8(float* out, int iters) {
  float d[4][4] = {};
  uint32_t a = threadIdx.x, b = threadIdx.x * 3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4}, {%5}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3]) : "r"(a), "r"(b));
  float s = 0; for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kmov(float* out, int iters) {
  uint32_t x[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x[j]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = x[0] + x[1] + x[2] + x[3];
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148, iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    const char* nm[3] = {"m16n8k16", "m16n8k8", "movmatrix"};
    for (int w = 0; w < 3; ++w) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (w == 0) k16<<<sms, warps * 32>>>(o, iters);
        else if (w == 1) k8<<<sms, warps * 32>>>(o, iters);
        else kmov<<<sms, warps * 32>>>(o, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * warps * iters * 4;  // warp-instructions
        if (rep) printf("%-10s warps/SM=%2d: %.3f ms, %.2f warp-inst/clk/SM (at 1.965 GHz)\n", nm[w], warps, ms,
                        ops / sms / (ms * 1e-3 * 1.965e9));
      }
    }
  }
  return 0;
}

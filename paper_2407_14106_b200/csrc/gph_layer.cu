// The transformer layer around the attention: one pre-LN
// GPH block of the reference Trainer (proj/src/model.cpp:533-595 forward,
// :669-744 backward; LayerNorm proj/src/matrix.cpp:91-139, GELU
// model.cpp:20-32) on the device:
//
//   a = LN1(h); q, k, v = a W_{q,k,v} + b;  attn = SparseAttention(q, k, v)
//   h += attn W_o + b_o;  b = LN2(h);  u = b W_ff1 + b_ff1
//   h += gelu(u) W_ff2 + b_ff2
//
// The projections are cuBLAS GEMMs (library GEMMs; the residual adds ride on
// beta = 1, the bias broadcasts are pre-filled rows); LayerNorm (one warp per
// row, statistics in the accumulate type), bias+GELU and the column sums of
// the bias gradients (per-CTA partials + a fixed-order pass: deterministic)
// are kernels here; the attention is the plan's sparse kernels (q and k share
// one [S x 2d] buffer so one leading dimension serves both, as the C ABI
// wants). Dropout is off (the timed / parity configuration of the Trainer).
// dtype: f64 (conformance), f32, bf16 (activations and weights bf16, fp32
// accumulation and statistics, fp32 parameter gradients).
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define GCU(x)                                                                                        \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)
#define GBL(x)                                                                                            \
  do {                                                                                                    \
    cublasStatus_t s_ = (x);                                                                              \
    if (s_ != CUBLAS_STATUS_SUCCESS) return set_error(GTE_CUDA, "cuBLAS error " + std::to_string((int)s_)); \
  } while (0)
#define GTRY(x)          \
  do {                   \
    int rc_ = (x);       \
    if (rc_) return rc_; \
  } while (0)

namespace {

constexpr double kLnEps = 1e-6;  // matrix.cpp:87
constexpr int kColParts = 148;   // CTAs of the column-sum partial pass

template <typename T> struct AccT { using type = float; };
template <> struct AccT<double> { using type = double; };
__device__ __forceinline__ float to_a(float x) { return x; }
__device__ __forceinline__ double to_a(double x) { return x; }
__device__ __forceinline__ float to_a(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_a(typename AccT<T>::type x);
template <> __device__ __forceinline__ float from_a<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_a<double>(double x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_a<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

template <typename A>
__device__ __forceinline__ A warp_sum(A x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// LayerNorm rows (matrix.cpp:91-113): out = (x - mu) * inv * scale + shift;
// keeps mu, inv per row for the backward (which recomputes the normalised x)
template <typename T>
__global__ void ln_fwd_kernel(const T* __restrict__ x, int64_t S, int d, const typename AccT<T>::type* __restrict__ sc,
                              const typename AccT<T>::type* __restrict__ sh, T* __restrict__ out,
                              typename AccT<T>::type* __restrict__ mu_o, typename AccT<T>::type* __restrict__ inv_o) {
  using A = typename AccT<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= S) return;
  const T* xr = x + r * d;
  A s = 0;
  for (int j = lane; j < d; j += 32) s += to_a(xr[j]);
  const A mu = warp_sum(s) / A(d);
  A v = 0;
  for (int j = lane; j < d; j += 32) {
    const A t = to_a(xr[j]) - mu;
    v += t * t;
  }
  const A inv = A(1) / sqrt(warp_sum(v) / A(d) + A(kLnEps));
  for (int j = lane; j < d; j += 32) out[r * d + j] = from_a<T>((to_a(xr[j]) - mu) * inv * sc[j] + sh[j]);
  if (lane == 0) {
    mu_o[r] = mu;
    inv_o[r] = inv;
  }
}

// LayerNorm backward (matrix.cpp:116-139): dx += inv (dn - mean(dn) - nh mean(dn nh)),
// dn = dout * scale; per-CTA partial sums of dscale = sum dout*nh, dshift = sum dout
template <typename T>
__global__ void ln_bwd_kernel(const T* __restrict__ dout, const T* __restrict__ x, int64_t S, int d,
                              const typename AccT<T>::type* __restrict__ sc, const typename AccT<T>::type* __restrict__ mu_i,
                              const typename AccT<T>::type* __restrict__ inv_i, T* __restrict__ dx,
                              typename AccT<T>::type* __restrict__ part /* [gridDim.x][2][d] */) {
  using A = typename AccT<T>::type;
  extern __shared__ unsigned char ln_smem[];
  A* ps = reinterpret_cast<A*>(ln_smem);  // [warps][2][d]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x / 32;
  A* mine = ps + (size_t)warp * 2 * d;
  for (int j = lane; j < 2 * d; j += 32) mine[j] = 0;
  for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < S; r += (int64_t)gridDim.x * nw) {
    const A mu = mu_i[r], inv = inv_i[r];
    A m1 = 0, m2 = 0;
    for (int j = lane; j < d; j += 32) {
      const A nh = (to_a(x[r * d + j]) - mu) * inv, g = to_a(dout[r * d + j]);
      const A dn = g * sc[j];
      mine[j] += g * nh;
      mine[d + j] += g;
      m1 += dn;
      m2 += dn * nh;
    }
    m1 = warp_sum(m1) / A(d);
    m2 = warp_sum(m2) / A(d);
    for (int j = lane; j < d; j += 32) {
      const A nh = (to_a(x[r * d + j]) - mu) * inv;
      const A dn = to_a(dout[r * d + j]) * sc[j];
      dx[r * d + j] = from_a<T>(to_a(dx[r * d + j]) + inv * (dn - m1 - nh * m2));
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 2 * d; j += blockDim.x) {  // warps in order
    A t = 0;
    for (int w = 0; w < nw; ++w) t += ps[(size_t)w * 2 * d + j];
    part[(size_t)blockIdx.x * 2 * d + j] = t;
  }
}

// column sums of a [S x n] matrix: per-CTA partials over row ranges
template <typename T>
__global__ void colsum_part_kernel(const T* __restrict__ m, int64_t S, int n, int64_t ld,
                                   typename AccT<T>::type* __restrict__ part /* [gridDim.x][n] */) {
  using A = typename AccT<T>::type;
  const int64_t r0 = S * blockIdx.x / gridDim.x, r1 = S * (blockIdx.x + 1) / gridDim.x;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    A s = 0;
    for (int64_t r = r0; r < r1; ++r) s += to_a(m[r * ld + j]);
    part[(size_t)blockIdx.x * n + j] = s;
  }
}

// out[j] += sum over parts (fixed order)
template <typename A>
__global__ void part_reduce_kernel(const A* __restrict__ part, int parts, int n, A* __restrict__ out, int64_t stride) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    A s = 0;
    for (int p = 0; p < parts; ++p) s += part[(size_t)p * stride + j];
    out[j] += s;
  }
}

// rows of y [S x n] (leading dim ld) = bias (broadcast)
template <typename T>
__global__ void fill_bias_kernel(T* __restrict__ y, int64_t S, int n, int64_t ld, const typename AccT<T>::type* __restrict__ b) {
  const int64_t total = S * n;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x)
    y[(x / n) * ld + x % n] = from_a<T>(b[x % n]);
}

// y += bias rows
template <typename T>
__global__ void add_bias_kernel(T* __restrict__ y, int64_t S, int n, const typename AccT<T>::type* __restrict__ b) {
  const int64_t total = S * n;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x)
    y[x] = from_a<T>(to_a(y[x]) + b[x % n]);
}

template <typename A>
__device__ __forceinline__ A gelu_f(A x) {  // model.cpp:20-24
  const A c = A(0.7978845608028654), a = A(0.044715);
  return A(0.5) * x * (A(1) + tanh(c * (x + a * x * x * x)));
}
template <typename A>
__device__ __forceinline__ A gelu_g(A x) {  // model.cpp:26-32
  const A c = A(0.7978845608028654), a = A(0.044715);
  const A t = tanh(c * (x + a * x * x * x));
  return A(0.5) * (A(1) + t) + A(0.5) * x * (A(1) - t * t) * c * (A(1) + A(3) * a * x * x);
}

template <typename T>
__global__ void gelu_fwd_kernel(const T* __restrict__ u, T* __restrict__ g, int64_t n) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    g[x] = from_a<T>(gelu_f(to_a(u[x])));
}
template <typename T>
__global__ void gelu_bwd_kernel(const T* __restrict__ u, T* __restrict__ dg_to_du, int64_t n) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    dg_to_du[x] = from_a<T>(to_a(dg_to_du[x]) * gelu_g(to_a(u[x])));
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

size_t es_of(int dt) { return dt == GTE_F64 ? 8 : dt == GTE_F32 ? 4 : 2; }
size_t as_of(int dt) { return dt == GTE_F64 ? 8 : 4; }

struct Buf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  ~Buf() { cudaFree(p); }
};

}  // namespace

struct gte_gph_layer {
  gte_ctx* ctx = nullptr;
  const gte_plan* plan = nullptr;
  int dtype = GTE_F32;
  int64_t S = 0, E = 0;
  int H = 0, d = 0, dh = 0, ffn = 0;
  cublasHandle_t blas = nullptr;
  gte_gph_params w{};
  // tape (forward activations kept for the backward)
  Buf h_in, a, qk, v, attn, lse, h_mid, b, u, g, mu1, inv1, mu2, inv2;
  // backward scratch
  Buf dqk, dv, dattn, dg, da, part;

  cudaStream_t st() const { return static_cast<cudaStream_t>(ctx_stream(ctx)); }

  // row-major C[M x N] = alpha op(A) op(B) + beta C; A, B of dtype, C of dtype (ct = 0) or
  // of the accumulate type (ct = 1: parameter gradients)
  int gemm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
           void* C, int64_t ldc, double beta, int ct = 0) {
    GBL(cublasSetStream(blas, st()));
    // column-major view: C^T = op(B)^T op(A)^T
    const cublasOperation_t oa = tb ? CUBLAS_OP_T : CUBLAS_OP_N, ob = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
    if (dtype == GTE_F64) {
      const double one = 1.0;
      GBL(cublasDgemm(blas, oa, ob, (int)N, (int)M, (int)K, &one, static_cast<const double*>(B), (int)ldb,
                      static_cast<const double*>(A), (int)lda, &beta, static_cast<double*>(C), (int)ldc));
    } else {
      const float one = 1.f, bf = (float)beta;
      const cudaDataType_t in = dtype == GTE_F32 ? CUDA_R_32F : CUDA_R_16BF;
      const cudaDataType_t out = ct ? CUDA_R_32F : in;
      GBL(cublasGemmEx(blas, oa, ob, (int)N, (int)M, (int)K, &one, B, in, (int)ldb, A, in, (int)lda, &bf, C, out,
                       (int)ldc, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT));
    }
    ctx_launch_counter(ctx) += 1;
    return GTE_OK;
  }
};

namespace {

template <typename T>
int ln_fwd(gte_gph_layer* L, const void* x, const void* sc, const void* sh, void* out, Buf& mu, Buf& inv) {
  using A = typename AccT<T>::type;
  GCU(mu.ensure(sizeof(A) * L->S));
  GCU(inv.ensure(sizeof(A) * L->S));
  const int rows_per = 8;
  ln_fwd_kernel<T><<<(unsigned)((L->S + rows_per - 1) / rows_per), 32 * rows_per, 0, L->st()>>>(
      static_cast<const T*>(x), L->S, L->d, static_cast<const A*>(sc), static_cast<const A*>(sh), static_cast<T*>(out),
      static_cast<A*>(mu.p), static_cast<A*>(inv.p));
  GCU(cudaGetLastError());
  ctx_launch_counter(L->ctx) += 1;
  return GTE_OK;
}

template <typename T>
int ln_bwd(gte_gph_layer* L, const void* dout, const void* x, const void* sc, Buf& mu, Buf& inv, void* dx,
           void* dscale, void* dshift) {
  using A = typename AccT<T>::type;
  const int warps = 8, d = L->d;
  GCU(L->part.ensure(sizeof(A) * kColParts * 2 * d));
  const size_t smem = sizeof(A) * warps * 2 * d;
  if (smem > 48 * 1024) GCU(cudaFuncSetAttribute(ln_bwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ln_bwd_kernel<T><<<kColParts, 32 * warps, smem, L->st()>>>(
      static_cast<const T*>(dout), static_cast<const T*>(x), L->S, d, static_cast<const A*>(sc),
      static_cast<const A*>(mu.p), static_cast<const A*>(inv.p), static_cast<T*>(dx), static_cast<A*>(L->part.p));
  part_reduce_kernel<A><<<grid_of(d), 256, 0, L->st()>>>(static_cast<A*>(L->part.p), kColParts, d,
                                                           static_cast<A*>(dscale), 2 * d);
  part_reduce_kernel<A><<<grid_of(d), 256, 0, L->st()>>>(static_cast<A*>(L->part.p) + d, kColParts, d,
                                                           static_cast<A*>(dshift), 2 * d);
  GCU(cudaGetLastError());
  ctx_launch_counter(L->ctx) += 3;
  return GTE_OK;
}

template <typename T>
int colsum_add(gte_gph_layer* L, const void* m, int n, int64_t ld, void* out) {
  using A = typename AccT<T>::type;
  GCU(L->part.ensure(sizeof(A) * kColParts * n));
  colsum_part_kernel<T><<<kColParts, 256, 0, L->st()>>>(static_cast<const T*>(m), L->S, n, ld, static_cast<A*>(L->part.p));
  part_reduce_kernel<A><<<grid_of(n), 256, 0, L->st()>>>(static_cast<A*>(L->part.p), kColParts, n, static_cast<A*>(out), n);
  GCU(cudaGetLastError());
  ctx_launch_counter(L->ctx) += 2;
  return GTE_OK;
}

template <typename T>
int fwd_t(gte_gph_layer* L, void* h, const void* bias_vals) {
  using A = typename AccT<T>::type;
  const size_t es = sizeof(T);
  const int64_t S = L->S, d = L->d, f = L->ffn;
  cudaStream_t st = L->st();
  const gte_gph_params& w = L->w;
  GCU(L->h_in.ensure(es * S * d));
  GCU(L->a.ensure(es * S * d));
  GCU(L->qk.ensure(es * S * 2 * d));
  GCU(L->v.ensure(es * S * d));
  GCU(L->attn.ensure(es * S * d));
  GCU(L->lse.ensure(sizeof(A) * S * L->H));
  GCU(L->h_mid.ensure(es * S * d));
  GCU(L->b.ensure(es * S * d));
  GCU(L->u.ensure(es * S * f));
  GCU(L->g.ensure(es * S * f));
  GCU(cudaMemcpyAsync(L->h_in.p, h, es * S * d, cudaMemcpyDeviceToDevice, st));
  GTRY(ln_fwd<T>(L, h, w.ln1_scale, w.ln1_shift, L->a.p, L->mu1, L->inv1));
  // q | k into one [S x 2d] buffer, v apart (the attention's two leading dims)
  fill_bias_kernel<T><<<grid_of(S * d), 256, 0, st>>>(static_cast<T*>(L->qk.p), S, (int)d, 2 * d, static_cast<const A*>(w.b_q));
  fill_bias_kernel<T><<<grid_of(S * d), 256, 0, st>>>(static_cast<T*>(L->qk.p) + d, S, (int)d, 2 * d, static_cast<const A*>(w.b_k));
  fill_bias_kernel<T><<<grid_of(S * d), 256, 0, st>>>(static_cast<T*>(L->v.p), S, (int)d, d, static_cast<const A*>(w.b_v));
  GTRY(L->gemm(false, false, S, d, d, L->a.p, d, w.w_q, d, L->qk.p, 2 * d, 1.0));
  GTRY(L->gemm(false, false, S, d, d, L->a.p, d, w.w_k, d, static_cast<T*>(L->qk.p) + d, 2 * d, 1.0));
  GTRY(L->gemm(false, false, S, d, d, L->a.p, d, w.w_v, d, L->v.p, d, 1.0));
  GTRY(gte_sparse_attn_fwd(L->ctx, L->plan, L->dtype, L->H, L->dh, L->dh, L->qk.p, static_cast<T*>(L->qk.p) + d,
                           2 * d, L->v.p, d, bias_vals, nullptr, L->attn.p, L->lse.p, 0));
  // h += attn W_o + b_o
  add_bias_kernel<T><<<grid_of(S * d), 256, 0, st>>>(static_cast<T*>(h), S, (int)d, static_cast<const A*>(w.b_o));
  GTRY(L->gemm(false, false, S, d, d, L->attn.p, d, w.w_o, d, h, d, 1.0));
  GCU(cudaMemcpyAsync(L->h_mid.p, h, es * S * d, cudaMemcpyDeviceToDevice, st));
  GTRY(ln_fwd<T>(L, h, w.ln2_scale, w.ln2_shift, L->b.p, L->mu2, L->inv2));
  fill_bias_kernel<T><<<grid_of(S * f), 256, 0, st>>>(static_cast<T*>(L->u.p), S, (int)f, f, static_cast<const A*>(w.b_ff1));
  GTRY(L->gemm(false, false, S, f, d, L->b.p, d, w.w_ff1, f, L->u.p, f, 1.0));
  gelu_fwd_kernel<T><<<grid_of(S * f), 256, 0, st>>>(static_cast<const T*>(L->u.p), static_cast<T*>(L->g.p), S * f);
  add_bias_kernel<T><<<grid_of(S * d), 256, 0, st>>>(static_cast<T*>(h), S, (int)d, static_cast<const A*>(w.b_ff2));
  GTRY(L->gemm(false, false, S, d, f, L->g.p, f, w.w_ff2, d, h, d, 1.0));
  GCU(cudaGetLastError());
  ctx_launch_counter(L->ctx) += 7;
  return GTE_OK;
}

template <typename T>
int bwd_t(gte_gph_layer* L, void* dh, const void* bias_vals, const gte_gph_params& gr, void* dbias_vals) {
  using A = typename AccT<T>::type;
  const size_t es = sizeof(T);
  const int64_t S = L->S, d = L->d, f = L->ffn;
  cudaStream_t st = L->st();
  const gte_gph_params& w = L->w;
  GCU(L->dg.ensure(es * S * f));
  GCU(L->da.ensure(es * S * d));
  GCU(L->dattn.ensure(es * S * d));
  GCU(L->dqk.ensure(es * S * 2 * d));
  GCU(L->dv.ensure(es * S * d));
  // second residual: df = dh
  GTRY(L->gemm(true, false, f, d, S, L->g.p, f, dh, d, (gr.w_ff2), d, 1.0, 1));
  GTRY(colsum_add<T>(L, dh, (int)d, d, (gr.b_ff2)));
  GTRY(L->gemm(false, true, S, f, d, dh, d, w.w_ff2, d, L->dg.p, f, 0.0));
  gelu_bwd_kernel<T><<<grid_of(S * f), 256, 0, st>>>(static_cast<const T*>(L->u.p), static_cast<T*>(L->dg.p), S * f);
  GTRY(L->gemm(true, false, d, f, S, L->b.p, d, L->dg.p, f, (gr.w_ff1), f, 1.0, 1));
  GTRY(colsum_add<T>(L, L->dg.p, (int)f, f, (gr.b_ff1)));
  GTRY(L->gemm(false, true, S, d, f, L->dg.p, f, w.w_ff1, f, L->da.p, d, 0.0));
  GTRY(ln_bwd<T>(L, L->da.p, L->h_mid.p, w.ln2_scale, L->mu2, L->inv2, dh, (gr.ln2_scale),
                 (gr.ln2_shift)));
  // first residual: do = dh
  GTRY(L->gemm(true, false, d, d, S, L->attn.p, d, dh, d, (gr.w_o), d, 1.0, 1));
  GTRY(colsum_add<T>(L, dh, (int)d, d, (gr.b_o)));
  GTRY(L->gemm(false, true, S, d, d, dh, d, w.w_o, d, L->dattn.p, d, 0.0));
  GTRY(gte_sparse_attn_bwd(L->ctx, L->plan, L->dtype, L->H, L->dh, L->dh, L->qk.p, static_cast<T*>(L->qk.p) + d,
                           2 * d, L->v.p, d, L->attn.p, L->lse.p, L->dattn.p, bias_vals, nullptr, L->dqk.p,
                           static_cast<T*>(L->dqk.p) + d, L->dv.p, dbias_vals));
  GTRY(L->gemm(true, false, d, d, S, L->a.p, d, L->dqk.p, 2 * d, (gr.w_q), d, 1.0, 1));
  GTRY(L->gemm(true, false, d, d, S, L->a.p, d, static_cast<T*>(L->dqk.p) + d, 2 * d, (gr.w_k), d, 1.0, 1));
  GTRY(L->gemm(true, false, d, d, S, L->a.p, d, L->dv.p, d, (gr.w_v), d, 1.0, 1));
  GTRY(colsum_add<T>(L, L->dqk.p, (int)d, 2 * d, (gr.b_q)));
  GTRY(colsum_add<T>(L, static_cast<T*>(L->dqk.p) + d, (int)d, 2 * d, (gr.b_k)));
  GTRY(colsum_add<T>(L, L->dv.p, (int)d, d, (gr.b_v)));
  GTRY(L->gemm(false, true, S, d, d, L->dqk.p, 2 * d, w.w_q, d, L->da.p, d, 0.0));
  GTRY(L->gemm(false, true, S, d, d, static_cast<T*>(L->dqk.p) + d, 2 * d, w.w_k, d, L->da.p, d, 1.0));
  GTRY(L->gemm(false, true, S, d, d, L->dv.p, d, w.w_v, d, L->da.p, d, 1.0));
  GTRY(ln_bwd<T>(L, L->da.p, L->h_in.p, w.ln1_scale, L->mu1, L->inv1, dh, (gr.ln1_scale),
                 (gr.ln1_shift)));
  GCU(cudaGetLastError());
  ctx_launch_counter(L->ctx) += 1;
  return GTE_OK;
}

}  // namespace

extern "C" {

int gte_gph_layer_create(gte_ctx* ctx, const gte_plan* plan, int dtype, int heads, int hidden, int ffn,
                         gte_gph_layer** out) {
  if (dtype != GTE_F64 && dtype != GTE_F32 && dtype != GTE_BF16) return set_error(GTE_CONFIG, "layer: bad dtype");
  if (heads < 1 || hidden % heads != 0) return set_error(GTE_CONFIG, "layer: hidden dim not divisible by head count");
  if (ffn < 1) return set_error(GTE_CONFIG, "layer: ffn dim must be >= 1");
  int64_t rows = 0, nnz = 0;
  GTRY(gte_plan_shape(plan, &rows, &nnz, nullptr, nullptr));
  auto* L = new gte_gph_layer();
  L->ctx = ctx;
  L->plan = plan;
  L->dtype = dtype;
  L->S = rows;
  L->E = nnz;
  L->H = heads;
  L->d = hidden;
  L->dh = hidden / heads;
  L->ffn = ffn;
  if (cublasCreate(&L->blas) != CUBLAS_STATUS_SUCCESS) {
    delete L;
    return set_error(GTE_CUDA, "layer: cublasCreate failed");
  }
  *out = L;
  return GTE_OK;
}

int gte_gph_layer_destroy(gte_gph_layer* L) {
  if (!L) return GTE_OK;
  cublasDestroy(L->blas);
  delete L;
  return GTE_OK;
}

int gte_gph_layer_set_params(gte_gph_layer* L, const gte_gph_params* p) {
  L->w = *p;
  return GTE_OK;
}

int gte_gph_layer_fwd(gte_gph_layer* L, void* h, const void* bias_vals) {
  switch (L->dtype) {
    case GTE_F64: return fwd_t<double>(L, h, bias_vals);
    case GTE_F32: return fwd_t<float>(L, h, bias_vals);
    default: return fwd_t<__nv_bfloat16>(L, h, bias_vals);
  }
}

int gte_gph_layer_bwd(gte_gph_layer* L, void* dh, const void* bias_vals, const gte_gph_params* grads, void* dbias_vals) {
  switch (L->dtype) {
    case GTE_F64: return bwd_t<double>(L, dh, bias_vals, *grads, dbias_vals);
    case GTE_F32: return bwd_t<float>(L, dh, bias_vals, *grads, dbias_vals);
    default: return bwd_t<__nv_bfloat16>(L, dh, bias_vals, *grads, dbias_vals);
  }
}

}  // extern "C"

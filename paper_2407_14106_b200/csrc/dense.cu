// Dense (all-pairs) attention, flash-style: the reference's dense_attention /
// dense_attention_backward (proj/src/attention.cpp:46-94, 174-239) and the
// Trainer's dense epoch semantics (proj/src/model.cpp:395-405: real rows
// attend exactly the real columns [0, s_real), pad rows only themselves)
// without materialising the S x S pattern.
//
// Forward: a CTA owns BR query rows of one head; K/V tiles of BC columns are
// staged in shared memory (accumulate type) and every thread runs an online
// softmax over its RPT rows, reading each staged K/V row once per RPT rows
// (register blocking). Scores, LSE, outputs in the accumulate type (f64 for
// the conformance mode, f32 otherwise); natural exp in f64, ex2 in the log2
// domain in f32.
//
// Backward, atomic-free (two passes, like the sparse kernels):
//   rows: per row and head, delta = sum_j w_j dw_j (= dO . O), recompute p,
//         dQ, and dbias[i][j] = sum over heads of ds (RMW of the row's own
//         entries, heads in order 0..H-1);
//   cols: per column and head, recompute p and ds for every real row: dK, dV.
// Pad rows (>= s_real) attend only themselves: out = m * v_i exactly, no
// gradient through the score (the sparse kernels' degree-1 rule).
//
// Bounds: dh <= 64. The S x S bias (shared by heads) and the head-major
// [H x S x S] weight_mult are optional, as in the reference API.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
cudaError_t launch_dense_tc_fwd(int64_t S, int64_t s_real, int H, int dk, int dv, const void* q, const void* k,
                                int64_t ldq, const void* v, int64_t ldv, const void* bias, const void* wmult,
                                void* out, void* lse, cudaStream_t st);
cudaError_t launch_dense_tc_bwd(int64_t S, int64_t s_real, int H, int dk, int dv, const void* q, const void* k,
                                int64_t ldq, const void* v, int64_t ldv, const void* out, const void* lse,
                                const void* dout, const void* bias, void* dq, void* dk_out, void* dv_out,
                                float* delta_ws, cudaStream_t st);
void* ctx_scratch(gte_ctx* c, size_t bytes);
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define DCUDA(expr)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                 \
  } while (0)

namespace {

constexpr int kBR = 128;  // rows per CTA (threads x RPT)
constexpr int kBC = 32;   // staged columns per tile

template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float ld_acc(const float* p) { return __ldg(p); }
__device__ __forceinline__ double ld_acc(const double* p) { return __ldg(p); }
__device__ __forceinline__ float ld_acc(const __nv_bfloat16* p) { return __bfloat162float(p[0]); }
__device__ __forceinline__ void st_val(float* p, float x) { *p = x; }
__device__ __forceinline__ void st_val(double* p, double x) { *p = x; }
__device__ __forceinline__ void st_val(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

template <typename A> struct DMath;
template <> struct DMath<float> {
  static constexpr float kL = 1.4426950408889634f;  // scores kept in log2 units
  __device__ static float ex(float x) { return exp2f(x); }
  __device__ static float lg(float x) { return log2f(x); }
  __device__ static float ninf() { return -INFINITY; }
};
template <> struct DMath<double> {
  static constexpr double kL = 1.0;
  __device__ static double ex(double x) { return exp(x); }
  __device__ static double lg(double x) { return log(x); }
  __device__ static double ninf() { return -INFINITY; }
};

constexpr int kMaxBuckets = 12;  // SPD buckets of the bucket-bias form (spd_cap <= 10; Trainer default 8)

struct DenseArgs {
  int64_t S, s_real;
  int H, dk, dv;
  int64_t ldq, ldv;
  const void *q, *k, *v, *o, *dout;
  const void* bias;   // A [S*S] or null
  // bucket-bias form (the Trainer's dense epoch, model.cpp:395-423, 520-523):
  // bias[r][c] = table[bucket[r][c]]; the backward reduces dbias per bucket
  const uint8_t* bucket;  // [S*S] or null
  const void* table;      // A [nb]
  int nb;
  void* dtable_part;      // A [gridDim.x][nb] (backward rows pass)
  const void* wmult;  // A [H*S*S] or null
  void *out, *lse, *dq, *dk_out, *dv_out;
  void* dbias;  // A [S*S] or null (backward)
  double scale;
};

// Stage columns [c0, c0 + n) of head h: Ks[c][t] (t < dk), Vs[c][t] (t < dv).
template <typename T, typename A, int DH>
__device__ __forceinline__ void stage_kv(const DenseArgs& a, int h, int64_t c0, int n, A (*Ks)[DH], A (*Vs)[DH],
                                         const T* K, const T* V) {
  for (int x = threadIdx.x; x < kBC * DH; x += blockDim.x) {
    const int c = x / DH, t = x % DH;
    A kv = 0, vv = 0;
    if (c < n) {
      if (t < a.dk) kv = ld_acc(K + (c0 + c) * a.ldq + (int64_t)h * a.dk + t);
      if (t < a.dv) vv = ld_acc(V + (c0 + c) * a.ldv + (int64_t)h * a.dv + t);
    }
    Ks[c][t] = kv;
    Vs[c][t] = vv;
  }
}

// -------------------------------------------------------------------- fwd
template <typename T, int DH, int RPT>
__global__ void __launch_bounds__(kBR / RPT) dense_fwd_kernel(DenseArgs a) {
  using A = typename Acc<T>::type;
  using M = DMath<A>;
  __shared__ A Ks[kBC][DH], Vs[kBC][DH], Tb[kMaxBuckets];
  const int h = blockIdx.y;
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const A* bias = static_cast<const A*>(a.bias);
  const uint8_t* bk = a.bucket;
  if (threadIdx.x < a.nb) Tb[threadIdx.x] = static_cast<const A*>(a.table)[threadIdx.x];
  const A* wm = static_cast<const A*>(a.wmult);
  T* O = static_cast<T*>(a.out);
  A* LSE = static_cast<A*>(a.lse);
  const A scale_l = A(a.scale) * M::kL;
  const int64_t r0 = (int64_t)blockIdx.x * kBR + threadIdx.x * RPT;

  A q[RPT][DH], acc[RPT][DH], m[RPT], l[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t r = r0 + u;
#pragma unroll
    for (int t = 0; t < DH; ++t) {
      q[u][t] = (r < a.s_real && t < a.dk) ? ld_acc(Q + r * a.ldq + (int64_t)h * a.dk + t) : A(0);
      acc[u][t] = 0;
    }
    m[u] = M::ninf();
    l[u] = 0;
  }
  for (int64_t c0 = 0; c0 < a.s_real; c0 += kBC) {
    const int n = (int)(a.s_real - c0 < kBC ? a.s_real - c0 : kBC);
    __syncthreads();
    stage_kv<T, A, DH>(a, h, c0, n, Ks, Vs, K, V);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = r0 + u;
      if (r >= a.s_real) continue;
      A s[kBC];
      A mx = M::ninf();
#pragma unroll
      for (int c = 0; c < kBC; ++c) {
        A d = 0;
#pragma unroll
        for (int t = 0; t < DH; ++t) d += q[u][t] * Ks[c][t];
        A x = d * scale_l;
        if (bias && c < n) x += bias[r * a.S + c0 + c] * M::kL;
        if (bk && c < n) x += Tb[bk[r * a.S + c0 + c]] * M::kL;
        s[c] = c < n ? x : M::ninf();
        mx = mx > s[c] ? mx : s[c];
      }
      const A mn = m[u] > mx ? m[u] : mx;
      const A corr = M::ex(m[u] - mn);
      l[u] *= corr;
#pragma unroll
      for (int t = 0; t < DH; ++t) acc[u][t] *= corr;
#pragma unroll
      for (int c = 0; c < kBC; ++c) {
        A p = M::ex(s[c] - mn);
        l[u] += p;
        if (wm && c < n) p *= wm[((int64_t)h * a.S + r) * a.S + c0 + c];
#pragma unroll
        for (int t = 0; t < DH; ++t) acc[u][t] += p * Vs[c][t];
      }
      m[u] = mn;
    }
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t r = r0 + u;
    if (r >= a.S) continue;
    if (r < a.s_real) {
      const A inv = A(1) / l[u];
#pragma unroll
      for (int t = 0; t < DH; ++t)
        if (t < a.dv) st_val(O + r * a.ldv + (int64_t)h * a.dv + t, acc[u][t] * inv);
      LSE[r * a.H + h] = m[u] + M::lg(l[u]);
    } else {  // pad row: attends only itself (model.cpp:400-403), out = m * v_r exactly
      const A mult = wm ? wm[((int64_t)h * a.S + r) * a.S + r] : A(1);
      for (int t = 0; t < a.dv; ++t) {
        const A vv = ld_acc(V + r * a.ldv + (int64_t)h * a.dv + t);
        st_val(O + r * a.ldv + (int64_t)h * a.dv + t, mult * vv);
      }
      LSE[r * a.H + h] = 0;  // unused (no score gradient)
    }
  }
}

// ------------------------------------------------------------- bwd rows
// dQ and dbias (heads in order inside the thread: dbias RMW is race-free)
template <typename T, int DH, int RPT>
__global__ void __launch_bounds__(kBR / RPT) dense_bwd_rows_kernel(DenseArgs a) {
  using A = typename Acc<T>::type;
  using M = DMath<A>;
  __shared__ A Ks[kBC][DH], Vs[kBC][DH], Tb[kMaxBuckets];
  __shared__ A Dt[kBR / RPT][kMaxBuckets];  // per-thread table gradient (fixed-order reduction below)
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* O = static_cast<const T*>(a.o);
  const T* DO = static_cast<const T*>(a.dout);
  const A* bias = static_cast<const A*>(a.bias);
  const uint8_t* bk = a.bucket;
  if (threadIdx.x < a.nb) Tb[threadIdx.x] = static_cast<const A*>(a.table)[threadIdx.x];
  for (int b = 0; b < kMaxBuckets; ++b) Dt[threadIdx.x][b] = 0;
  const A* wm = static_cast<const A*>(a.wmult);
  const A* LSE = static_cast<const A*>(a.lse);
  T* DQ = static_cast<T*>(a.dq);
  A* DB = static_cast<A*>(a.dbias);
  const A scale_l = A(a.scale) * M::kL;
  const int64_t r0 = (int64_t)blockIdx.x * kBR + threadIdx.x * RPT;

  for (int h = 0; h < a.H; ++h) {
    A q[RPT][DH], dd[RPT][DH], dq[RPT][DH], lse[RPT], delta[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = r0 + u;
      const bool real = r < a.s_real;
      A dl = 0;
#pragma unroll
      for (int t = 0; t < DH; ++t) {
        q[u][t] = (real && t < a.dk) ? ld_acc(Q + r * a.ldq + (int64_t)h * a.dk + t) : A(0);
        dd[u][t] = (real && t < a.dv) ? ld_acc(DO + r * a.ldv + (int64_t)h * a.dv + t) : A(0);
        const A oo = (real && t < a.dv) ? ld_acc(O + r * a.ldv + (int64_t)h * a.dv + t) : A(0);
        dl += dd[u][t] * oo;
        dq[u][t] = 0;
      }
      delta[u] = dl;
      lse[u] = real ? LSE[r * a.H + h] : A(0);
    }
    for (int64_t c0 = 0; c0 < a.s_real; c0 += kBC) {
      const int n = (int)(a.s_real - c0 < kBC ? a.s_real - c0 : kBC);
      __syncthreads();
      stage_kv<T, A, DH>(a, h, c0, n, Ks, Vs, K, V);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = r0 + u;
        if (r >= a.s_real) continue;
#pragma unroll 4
        for (int c = 0; c < n; ++c) {
          A d = 0, dw = 0;
#pragma unroll
          for (int t = 0; t < DH; ++t) {
            d += q[u][t] * Ks[c][t];
            dw += dd[u][t] * Vs[c][t];
          }
          A x = d * scale_l;
          if (bias) x += bias[r * a.S + c0 + c] * M::kL;
          const int bkt = bk ? bk[r * a.S + c0 + c] : 0;
          if (bk) x += Tb[bkt] * M::kL;
          const A p = M::ex(x - lse[u]);
          if (wm) dw *= wm[((int64_t)h * a.S + r) * a.S + c0 + c];
          const A ds = p * (dw - delta[u]);
          if (bk) Dt[threadIdx.x][bkt] += ds;
#pragma unroll
          for (int t = 0; t < DH; ++t) dq[u][t] += ds * Ks[c][t];
          if (DB) {
            A* db = DB + r * a.S + c0 + c;
            *db = h == 0 ? ds : *db + ds;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = r0 + u;
      if (r >= a.S) continue;
      const bool real = r < a.s_real;
#pragma unroll
      for (int t = 0; t < DH; ++t)
        if (t < a.dk) st_val(DQ + r * a.ldq + (int64_t)h * a.dk + t, real ? dq[u][t] * A(a.scale) : A(0));
    }
  }
  if (bk) {  // this CTA's table gradient: threads summed in index order
    __syncthreads();
    if (threadIdx.x < a.nb) {
      A g = 0;
      for (int t = 0; t < (int)blockDim.x; ++t) g += Dt[t][threadIdx.x];
      static_cast<A*>(a.dtable_part)[(int64_t)blockIdx.x * a.nb + threadIdx.x] = g;
    }
  }
}

// dtable[b] = sum over the rows pass's CTAs of their partials, in CTA order
template <typename A>
__global__ void dtable_reduce_kernel(const A* __restrict__ part, int nparts, int nb, A* __restrict__ out) {
  const int b = threadIdx.x;
  if (b >= nb) return;
  A g = 0;
  for (int x = 0; x < nparts; ++x) g += part[(int64_t)x * nb + b];
  out[b] = g;
}

// ------------------------------------------------------------- bwd cols
template <typename T, int DH, int RPT>
__global__ void __launch_bounds__(kBR / RPT) dense_bwd_cols_kernel(DenseArgs a) {
  using A = typename Acc<T>::type;
  using M = DMath<A>;
  __shared__ A Qs[kBC][DH], Ds[kBC][DH], Ls[kBC], Dl[kBC], Tb[kMaxBuckets];
  const int h = blockIdx.y;
  const uint8_t* bk = a.bucket;
  if (threadIdx.x < a.nb) Tb[threadIdx.x] = static_cast<const typename Acc<T>::type*>(a.table)[threadIdx.x];
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* O = static_cast<const T*>(a.o);
  const T* DO = static_cast<const T*>(a.dout);
  const A* bias = static_cast<const A*>(a.bias);
  const A* wm = static_cast<const A*>(a.wmult);
  const A* LSE = static_cast<const A*>(a.lse);
  T* DK = static_cast<T*>(a.dk_out);
  T* DV = static_cast<T*>(a.dv_out);
  const A scale_l = A(a.scale) * M::kL;
  const int64_t c00 = (int64_t)blockIdx.x * kBR + threadIdx.x * RPT;

  A kj[RPT][DH], vj[RPT][DH], gk[RPT][DH], gv[RPT][DH];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t c = c00 + u;
    const bool real = c < a.s_real;
#pragma unroll
    for (int t = 0; t < DH; ++t) {
      kj[u][t] = (real && t < a.dk) ? ld_acc(K + c * a.ldq + (int64_t)h * a.dk + t) : A(0);
      vj[u][t] = (real && t < a.dv) ? ld_acc(V + c * a.ldv + (int64_t)h * a.dv + t) : A(0);
      gk[u][t] = gv[u][t] = 0;
    }
  }
  for (int64_t i0 = 0; i0 < a.s_real; i0 += kBC) {
    const int n = (int)(a.s_real - i0 < kBC ? a.s_real - i0 : kBC);
    __syncthreads();
    for (int x = threadIdx.x; x < kBC * DH; x += blockDim.x) {
      const int i = x / DH, t = x % DH;
      A qv = 0, dv_ = 0;
      if (i < n) {
        if (t < a.dk) qv = ld_acc(Q + (i0 + i) * a.ldq + (int64_t)h * a.dk + t);
        if (t < a.dv) dv_ = ld_acc(DO + (i0 + i) * a.ldv + (int64_t)h * a.dv + t);
      }
      Qs[i][t] = qv;
      Ds[i][t] = dv_;
    }
    for (int i = threadIdx.x; i < kBC; i += blockDim.x) {
      A ls = 0, dl = 0;
      if (i < n) {
        ls = LSE[(i0 + i) * a.H + h];
        for (int t = 0; t < a.dv; ++t)
          dl += ld_acc(DO + (i0 + i) * a.ldv + (int64_t)h * a.dv + t) * ld_acc(O + (i0 + i) * a.ldv + (int64_t)h * a.dv + t);
      }
      Ls[i] = ls;
      Dl[i] = dl;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t c = c00 + u;
      if (c >= a.s_real) continue;
#pragma unroll 4
      for (int i = 0; i < n; ++i) {
        A d = 0, dw = 0;
#pragma unroll
        for (int t = 0; t < DH; ++t) {
          d += Qs[i][t] * kj[u][t];
          dw += Ds[i][t] * vj[u][t];
        }
        A x = d * scale_l;
        const int64_t r = i0 + i;
        if (bias) x += bias[r * a.S + c] * M::kL;
        if (bk) x += Tb[bk[r * a.S + c]] * M::kL;
        const A p = M::ex(x - Ls[i]);
        A pw = p;
        if (wm) {
          const A mult = wm[((int64_t)h * a.S + r) * a.S + c];
          dw *= mult;
          pw = p * mult;
        }
        const A ds = p * (dw - Dl[i]);
#pragma unroll
        for (int t = 0; t < DH; ++t) {
          gk[u][t] += ds * Qs[i][t];
          gv[u][t] += pw * Ds[i][t];
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t c = c00 + u;
    if (c >= a.S) continue;
    if (c < a.s_real) {
#pragma unroll
      for (int t = 0; t < DH; ++t) {
        if (t < a.dk) st_val(DK + c * a.ldq + (int64_t)h * a.dk + t, gk[u][t] * A(a.scale));
        if (t < a.dv) st_val(DV + c * a.ldv + (int64_t)h * a.dv + t, gv[u][t]);
      }
    } else {  // pad column: only its own (pad) row attends, p = 1: dV = m * dO, dK = 0
      const A mult = wm ? wm[((int64_t)h * a.S + c) * a.S + c] : A(1);
      for (int t = 0; t < a.dk; ++t) st_val(DK + c * a.ldq + (int64_t)h * a.dk + t, A(0));
      for (int t = 0; t < a.dv; ++t)
        st_val(DV + c * a.ldv + (int64_t)h * a.dv + t, mult * ld_acc(DO + c * a.ldv + (int64_t)h * a.dv + t));
    }
  }
}

template <typename T, int DH>
cudaError_t launch_dh(int which, const DenseArgs& a, cudaStream_t st) {
  constexpr int RPT = sizeof(T) == 8 ? 1 : (DH <= 16 ? 2 : 1);
  const dim3 grid((unsigned)((a.S + kBR - 1) / kBR), which == 1 ? 1u : (unsigned)a.H);
  const unsigned threads = kBR / RPT;
  if (which == 0)
    dense_fwd_kernel<T, DH, RPT><<<grid, threads, 0, st>>>(a);
  else if (which == 1)
    dense_bwd_rows_kernel<T, DH, RPT><<<grid, threads, 0, st>>>(a);
  else
    dense_bwd_cols_kernel<T, DH, RPT><<<grid, threads, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_t(int which, const DenseArgs& a, cudaStream_t st) {
  const int d = a.dk > a.dv ? a.dk : a.dv;
  if (d <= 8) return launch_dh<T, 8>(which, a, st);
  if (d <= 16) return launch_dh<T, 16>(which, a, st);
  if (d <= 32) return launch_dh<T, 32>(which, a, st);
  return launch_dh<T, 64>(which, a, st);
}

cudaError_t launch(int dtype, int which, const DenseArgs& a, cudaStream_t st) {
  switch (dtype) {
    case GTE_F64: return launch_t<double>(which, a, st);
    case GTE_F32: return launch_t<float>(which, a, st);
    default: return launch_t<__nv_bfloat16>(which, a, st);
  }
}

int check_args(int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, int64_t ldq, int64_t ldv) {
  if (dtype != GTE_F64 && dtype != GTE_F32 && dtype != GTE_BF16) return set_error(GTE_CONFIG, "dense_attention: bad dtype");
  if (dk < 1) return set_error(GTE_CONFIG, "attention: d_K must be >= 1");
  if (dv < 1) return set_error(GTE_CONFIG, "attention: d_V must be >= 1");
  if (dk > 64 || dv > 64) return set_error(GTE_CONFIG, "dense_attention: head dim > 64 unsupported");
  if (H < 1) return set_error(GTE_CONFIG, "dense_attention: heads must be >= 1");
  if (S < 0 || s_real < 0 || s_real > S) return set_error(GTE_CONFIG, "dense_attention: s_real must lie in [0, S]");
  if (ldq < (int64_t)H * dk || ldv < (int64_t)H * dv) return set_error(GTE_CONFIG, "dense_attention: leading dimension too small");
  return GTE_OK;
}

}  // namespace

extern "C" {

int gte_dense_attn_fwd(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                       const void* k, int64_t ldq, const void* v, int64_t ldv, const void* bias, const void* wmult,
                       void* out, void* lse) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  if (S == 0) return GTE_OK;
  DenseArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = q, a.k = k, a.v = v, a.bias = bias, a.wmult = wmult, a.out = out, a.lse = lse;
  a.scale = 1.0 / std::sqrt((double)dk);
  static const bool tc = [] {  // bf16: both GEMMs on tcgen05 (dense_tc.cu); GTE_DENSE_TC=0 -> CUDA cores
    const char* e = getenv("GTE_DENSE_TC");
    return !(e && e[0] == '0');
  }();
  if (dtype == GTE_BF16 && tc)
    DCUDA(launch_dense_tc_fwd(S, s_real, H, dk, dv, q, k, ldq, v, ldv, bias, wmult, out, lse,
                              (cudaStream_t)ctx_stream(ctx)));
  else
    DCUDA(launch(dtype, 0, a, (cudaStream_t)ctx_stream(ctx)));
  ctx_launch_counter(ctx) += 1;
  return GTE_OK;
}

int gte_dense_attn_bwd(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                       const void* k, int64_t ldq, const void* v, int64_t ldv, const void* out, const void* lse,
                       const void* dout, const void* bias, const void* wmult, void* dq, void* dk_out, void* dv_out,
                       void* dbias) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  if (S == 0) return GTE_OK;
  DenseArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = q, a.k = k, a.v = v, a.o = out, a.dout = dout, a.bias = bias, a.wmult = wmult, a.lse = const_cast<void*>(lse);
  a.dq = dq, a.dk_out = dk_out, a.dv_out = dv_out, a.dbias = dbias;
  a.scale = 1.0 / std::sqrt((double)dk);
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  static const bool tc = [] {  // bf16 without weight_mult / dbias: tcgen05 (dense_tc.cu)
    const char* e = getenv("GTE_DENSE_TC");
    return !(e && e[0] == '0');
  }();
  if (dtype == GTE_BF16 && tc && !wmult && !dbias) {
    float* ws = static_cast<float*>(ctx_scratch(ctx, sizeof(float) * (size_t)S * H));
    if (!ws) return set_error(GTE_CUDA, "dense_attention_backward: workspace allocation failed");
    DCUDA(launch_dense_tc_bwd(S, s_real, H, dk, dv, q, k, ldq, v, ldv, out, lse, dout, bias, dq, dk_out, dv_out, ws,
                              st));
    ctx_launch_counter(ctx) += 2;
    return GTE_OK;
  }
  if (dbias) DCUDA(cudaMemsetAsync(dbias, 0, sizeof(double) / (dtype == GTE_F64 ? 1 : 2) * (size_t)S * S, st));
  DCUDA(launch(dtype, 1, a, st));
  DCUDA(launch(dtype, 2, a, st));
  ctx_launch_counter(ctx) += 2;
  return GTE_OK;
}

// Bucket-bias form: the Trainer's dense epoch (model.cpp:395-423, 520-523)
// without an S x S float bias: bias[r][c] = table[buckets[r][c]] (uint8
// buckets from gte_dense_buckets), dtable[b] = sum of dbias over bucket b
// (fixed order: per-thread, per-CTA, then across CTAs). CUDA-core kernels for
// every dtype.
int gte_dense_attn_fwd_buckets(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv,
                               const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                               const uint8_t* buckets, const void* table, int64_t n_buckets, const void* wmult,
                               void* out, void* lse) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  if (!buckets || !table || n_buckets < 1 || n_buckets > kMaxBuckets)
    return set_error(GTE_CONFIG, "dense_attention: bucket bias needs 1.." + std::to_string(kMaxBuckets) + " buckets");
  if (S == 0) return GTE_OK;
  DenseArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = q, a.k = k, a.v = v, a.wmult = wmult, a.out = out, a.lse = lse;
  a.bucket = buckets, a.table = table, a.nb = (int)n_buckets;
  a.scale = 1.0 / std::sqrt((double)dk);
  DCUDA(launch(dtype, 0, a, (cudaStream_t)ctx_stream(ctx)));
  ctx_launch_counter(ctx) += 1;
  return GTE_OK;
}

int gte_dense_attn_bwd_buckets(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv,
                               const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv, const void* out,
                               const void* lse, const void* dout, const uint8_t* buckets, const void* table,
                               int64_t n_buckets, const void* wmult, void* dq, void* dk_out, void* dv_out,
                               void* dtable) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  if (!buckets || !table || n_buckets < 1 || n_buckets > kMaxBuckets)
    return set_error(GTE_CONFIG, "dense_attention: bucket bias needs 1.." + std::to_string(kMaxBuckets) + " buckets");
  if (S == 0) return GTE_OK;
  DenseArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = q, a.k = k, a.v = v, a.o = out, a.dout = dout, a.wmult = wmult, a.lse = const_cast<void*>(lse);
  a.dq = dq, a.dk_out = dk_out, a.dv_out = dv_out;
  a.bucket = buckets, a.table = table, a.nb = (int)n_buckets;
  a.scale = 1.0 / std::sqrt((double)dk);
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const int parts = (int)((S + kBR - 1) / kBR);
  const size_t as = dtype == GTE_F64 ? 8 : 4;
  void* part = nullptr;
  DCUDA(cudaMallocAsync(&part, as * (size_t)parts * n_buckets, st));
  a.dtable_part = part;
  DCUDA(launch(dtype, 1, a, st));
  DCUDA(launch(dtype, 2, a, st));
  if (dtype == GTE_F64)
    dtable_reduce_kernel<double><<<1, 32, 0, st>>>(static_cast<double*>(part), parts, (int)n_buckets,
                                                   static_cast<double*>(dtable));
  else
    dtable_reduce_kernel<float><<<1, 32, 0, st>>>(static_cast<float*>(part), parts, (int)n_buckets,
                                                  static_cast<float*>(dtable));
  DCUDA(cudaGetLastError());
  DCUDA(cudaFreeAsync(part, st));
  ctx_launch_counter(ctx) += 3;
  return GTE_OK;
}

// Host-buffer twins (synchronous): device buffers allocated per call, the
// stream synchronised before returning (the reference API is synchronous).
namespace {
struct HostDev {
  std::vector<void*> ptrs;
  ~HostDev() {
    for (void* p : ptrs) cudaFree(p);
  }
  void* put(const void* h, size_t bytes, cudaStream_t st, cudaError_t& e) {
    if (!h || e != cudaSuccess) return nullptr;
    void* d = nullptr;
    e = cudaMalloc(&d, bytes ? bytes : 16);
    if (e != cudaSuccess) return nullptr;
    ptrs.push_back(d);
    e = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    return d;
  }
  void* make(size_t bytes, cudaError_t& e) {
    if (e != cudaSuccess) return nullptr;
    void* d = nullptr;
    e = cudaMalloc(&d, bytes ? bytes : 16);
    if (e == cudaSuccess) ptrs.push_back(d);
    return d;
  }
};
size_t es_of(int dtype) { return dtype == GTE_F64 ? 8 : dtype == GTE_F32 ? 4 : 2; }
size_t as_of(int dtype) { return dtype == GTE_F64 ? 8 : 4; }
}  // namespace

int gte_dense_attn_fwd_host(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                            const void* k, const void* v, const void* bias, const void* wmult, void* out, void* lse) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, (int64_t)H * dk, (int64_t)H * dv);
  if (rc) return rc;
  if (S == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const size_t es = es_of(dtype), as = as_of(dtype), s2 = (size_t)S * S;
  cudaError_t e = cudaSuccess;
  HostDev m;
  void* dq = m.put(q, S * H * dk * es, st, e);
  void* dk_ = m.put(k, S * H * dk * es, st, e);
  void* dv_ = m.put(v, S * H * dv * es, st, e);
  void* db = m.put(bias, s2 * as, st, e);
  void* dw = m.put(wmult, s2 * H * as, st, e);
  void* dout = m.make(S * H * dv * es, e);
  void* dl = m.make(S * H * as, e);
  DCUDA(e);
  rc = gte_dense_attn_fwd(ctx, dtype, S, s_real, H, dk, dv, dq, dk_, (int64_t)H * dk, dv_, (int64_t)H * dv, db, dw,
                          dout, dl);
  if (rc) return rc;
  DCUDA(cudaMemcpyAsync(out, dout, S * H * dv * es, cudaMemcpyDeviceToHost, st));
  if (lse) DCUDA(cudaMemcpyAsync(lse, dl, S * H * as, cudaMemcpyDeviceToHost, st));
  DCUDA(cudaStreamSynchronize(st));
  return GTE_OK;
}

int gte_dense_attn_bwd_host(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                            const void* k, const void* v, const void* bias, const void* wmult, const void* dout,
                            void* dq, void* dk_out, void* dv_out, void* dbias) {
  int rc = check_args(dtype, S, s_real, H, dk, dv, (int64_t)H * dk, (int64_t)H * dv);
  if (rc) return rc;
  if (S == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const size_t es = es_of(dtype), as = as_of(dtype), s2 = (size_t)S * S;
  cudaError_t e = cudaSuccess;
  HostDev m;
  void* d_q = m.put(q, S * H * dk * es, st, e);
  void* d_k = m.put(k, S * H * dk * es, st, e);
  void* d_v = m.put(v, S * H * dv * es, st, e);
  void* d_b = m.put(bias, s2 * as, st, e);
  void* d_w = m.put(wmult, s2 * H * as, st, e);
  void* d_up = m.put(dout, S * H * dv * es, st, e);
  void* d_o = m.make(S * H * dv * es, e);
  void* d_l = m.make(S * H * as, e);
  void* g_q = m.make(S * H * dk * es, e);
  void* g_k = m.make(S * H * dk * es, e);
  void* g_v = m.make(S * H * dv * es, e);
  void* g_b = dbias ? m.make(s2 * as, e) : nullptr;
  DCUDA(e);
  rc = gte_dense_attn_fwd(ctx, dtype, S, s_real, H, dk, dv, d_q, d_k, (int64_t)H * dk, d_v, (int64_t)H * dv, d_b,
                          d_w, d_o, d_l);
  if (rc) return rc;
  rc = gte_dense_attn_bwd(ctx, dtype, S, s_real, H, dk, dv, d_q, d_k, (int64_t)H * dk, d_v, (int64_t)H * dv, d_o,
                          d_l, d_up, d_b, d_w, g_q, g_k, g_v, g_b);
  if (rc) return rc;
  DCUDA(cudaMemcpyAsync(dq, g_q, S * H * dk * es, cudaMemcpyDeviceToHost, st));
  DCUDA(cudaMemcpyAsync(dk_out, g_k, S * H * dk * es, cudaMemcpyDeviceToHost, st));
  DCUDA(cudaMemcpyAsync(dv_out, g_v, S * H * dv * es, cudaMemcpyDeviceToHost, st));
  if (dbias) DCUDA(cudaMemcpyAsync(dbias, g_b, s2 * as, cudaMemcpyDeviceToHost, st));
  DCUDA(cudaStreamSynchronize(st));
  return GTE_OK;
}

}  // extern "C"

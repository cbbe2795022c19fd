// Issue-efficient variant of the sparse graph-attention kernels for the
// aligned shapes that carry the benchmark configs (f32/bf16, head chunks that
// are a power-of-two number of 16-byte pieces, 16-byte aligned rows). Same
// math and outputs as the generic kernels in attn_sparse.cuh; the schedule and
// the instruction mix are what change (ncu showed the generic kernels issue-
// and latency-bound, not bandwidth-bound):
//
//   * each lane owns one 16-byte piece of one head of one neighbour
//     (VW = 16/sizeof(T) elements; LPH lanes per head; LPN = pow2(H)*LPH lanes
//     per neighbour; SLOTS = 32/LPN neighbours per warp step);
//   * the K/V (resp. Q/dO) gathers of a chunk of SLOTS*EPL edges are issued
//     back to back as 128-bit loads on clamped addresses, before any use;
//   * bf16 dot products run on FHFMA.BF16 (fma.rn.f32.bf16: bf16 operands,
//     fp32 accumulate — exact products, no unpacking), f32 ones on FFMA2
//     (fma.rn.f32x2), value accumulation on FFMA2;
//   * gather offsets are 32-bit (host guarantees rows*bytes < 2^32);
//   * Q/K/V finiteness is checked once per row on the row's own data (every
//     row is some warp's own row), not per gathered edge.
#pragma once

#include "attn_sparse.cuh"

#ifndef GTE_BF16_W
#define GTE_BF16_W 0
#endif

namespace gte_b200 {

// ---------------------------------------------------------------- packed math
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <typename T> struct Piece;

// f32: 4 elements per 16-byte piece
template <> struct Piece<float> {
  static constexpr int N = 4;
  // sum_t a_t*b_t as two FFMA2 lanes then one add
  __device__ __forceinline__ static float dot(const uint4& a, const uint4& b) {
    uint64_t p = ffma2(pk(__uint_as_float(a.x), __uint_as_float(a.y)), pk(__uint_as_float(b.x), __uint_as_float(b.y)),
                       pk(0.f, 0.f));
    p = ffma2(pk(__uint_as_float(a.z), __uint_as_float(a.w)), pk(__uint_as_float(b.z), __uint_as_float(b.w)), p);
    float x, y;
    upk(p, x, y);
    return __fadd_rn(x, y);
  }
  // acc[0..3] += w * x
  __device__ __forceinline__ static void axpy(float w, const uint4& x, float (&acc)[4]) {
    const uint64_t ww = pk(w, w);
    uint64_t lo = ffma2(ww, pk(__uint_as_float(x.x), __uint_as_float(x.y)), pk(acc[0], acc[1]));
    uint64_t hi = ffma2(ww, pk(__uint_as_float(x.z), __uint_as_float(x.w)), pk(acc[2], acc[3]));
    upk(lo, acc[0], acc[1]);
    upk(hi, acc[2], acc[3]);
  }
  __device__ __forceinline__ static void axpy_w(float w, const uint4& x, float (&acc)[4]) { axpy(w, x, acc); }
  __device__ __forceinline__ static float finite_probe(const uint4& x, float chk) {
    chk = __fmaf_rn(__uint_as_float(x.x), 0.f, chk);
    chk = __fmaf_rn(__uint_as_float(x.y), 0.f, chk);
    chk = __fmaf_rn(__uint_as_float(x.z), 0.f, chk);
    return __fmaf_rn(__uint_as_float(x.w), 0.f, chk);
  }
  __device__ __forceinline__ static uint4 pack(const float (&o)[4]) {
    return make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]), __float_as_uint(o[3]));
  }
};

// bf16: 8 elements per 16-byte piece
__device__ __forceinline__ float fma_bf16x2(uint32_t a, uint32_t b, float c) {
  float r;
  asm("{.reg .b16 al, ah, bl, bh; .reg .f32 t;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 t, al, bl, %3;\n\t"
      "fma.rn.f32.bf16 %0, ah, bh, t;}"
      : "=f"(r) : "r"(a), "r"(b), "f"(c));
  return r;
}

template <> struct Piece<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static float dot(const uint4& a, const uint4& b) {
    float s = fma_bf16x2(a.x, b.x, 0.f);
    s = fma_bf16x2(a.y, b.y, s);
    s = fma_bf16x2(a.z, b.z, s);
    return fma_bf16x2(a.w, b.w, s);
  }
  __device__ __forceinline__ static void axpy(float w, const uint4& x, float (&acc)[8]) {
    const uint64_t ww = pk(w, w);
    const uint32_t u[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t xv = pk(__uint_as_float(u[i] << 16), __uint_as_float(u[i] & 0xffff0000u));
      const uint64_t r = ffma2(ww, xv, pk(acc[2 * i], acc[2 * i + 1]));
      upk(r, acc[2 * i], acc[2 * i + 1]);
    }
  }
  // acc += w * x with w rounded to bf16 (GTE_BF16_W=1): 8 FHFMA.BF16 with
  // fp32 accumulation on the packed pairs, no unpacking. The weights are
  // softmax probabilities / score gradients, which flash attention also
  // rounds to bf16 before its P·V, dS·K, dS·Q products; 1 and 0 (degree-1
  // rows) stay exact.
  __device__ __forceinline__ static void axpy_w(float w, const uint4& x, float (&acc)[8]) {
#if GTE_BF16_W
    const unsigned short wb = __bfloat16_as_ushort(__float2bfloat16_rn(w));
    const uint32_t u[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
          "fma.rn.f32.bf16 %0, %3, l, %0;\n\tfma.rn.f32.bf16 %1, %3, h, %1;}"
          : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1]) : "r"(u[i]), "h"(wb));
#else
    axpy(w, x, acc);
#endif
  }
  __device__ __forceinline__ static float finite_probe(const uint4& x, float chk) {
    // a bf16 pair is non-finite iff one of its exponent fields is all ones
    const uint32_t u[4] = {x.x, x.y, x.z, x.w};
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) bad |= ((u[i] & 0x7f800000u) == 0x7f800000u) | ((u[i] & 0x7f80u) == 0x7f80u);
    return bad ? __int_as_float(0x7fc00000) : chk;
  }
  __device__ __forceinline__ static uint4 pack(const float (&o)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

__device__ __forceinline__ uint4 ldg16(const char* base, uint32_t off) {
  return __ldg(reinterpret_cast<const uint4*>(base + off));
}

template <int LPH>
__device__ __forceinline__ float head_sum(float x) {
#pragma unroll
  for (int o = 1; o < LPH; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

struct FastGeom {
  int lane, slot, hl, part, hcl;
  bool head_ok;
  uint32_t bo;  // byte offset of this lane's 16-byte piece inside a row
};

template <typename T, int LPH, int LPN>
__device__ __forceinline__ FastGeom fast_geom(int H, int dh) {
  FastGeom g;
  g.lane = lane_id();
  g.slot = g.lane / LPN;
  const int w = g.lane % LPN;
  g.hl = w / LPH;
  g.part = w % LPH;
  g.head_ok = g.hl < H;
  g.hcl = g.head_ok ? g.hl : 0;
  g.bo = g.head_ok ? (uint32_t)((g.hl * dh + g.part * Piece<T>::N) * (int)sizeof(T)) : 0u;
  return g;
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_fwd_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = float(p.scale) * M::kLogScale;
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  char* O = static_cast<char*>(p.out);
  float* __restrict__ LSE = static_cast<float*>(p.lse);
  const uint32_t rq = (uint32_t)(p.ldq * sizeof(T)), rv = (uint32_t)(p.ldv * sizeof(T));
  const WarpRange wr = warp_range(p);
  float chk_q = 0.f, chk_k = 0.f, chk_v = 0.f;

  for (int64_t i = wr.first; i < wr.last; i += wr.step) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    const uint4 q = ldg16(Q, (uint32_t)i * rq + g.bo);
    if (g.slot == 0 && g.head_ok) {  // own-row finiteness (attention.cpp:20-22)
      chk_q = P::finite_probe(q, chk_q);
      chk_k = P::finite_probe(ldg16(K, (uint32_t)i * rq + g.bo), chk_k);
      chk_v = P::finite_probe(ldg16(Vp, (uint32_t)i * rv + g.bo), chk_v);
    }
    float acc[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) acc[t] = 0.f;
    if (end == beg) {
      if (p.forbid_empty && g.lane == 0) atomicMin(p.err + 1, (int)i);
      if (g.slot == 0 && g.head_ok) {
        *reinterpret_cast<uint4*>(O + (uint32_t)i * rv + g.bo) = P::pack(acc);
        if (g.part == 0) LSE[i * p.H + g.hl] = M::neg_inf();
      }
      continue;
    }
    float m = M::neg_inf(), l = 0.f;
    for (int e0 = beg; e0 < end; e0 += CHUNK) {
      const int n = min(CHUNK, end - e0);
      const int my_col = g.lane < n ? __ldg(p.cols + e0 + g.lane) : (int)i;
      const float my_b = (bias && g.lane < n) ? __ldg(bias + e0 + g.lane) * M::kLogScale : 0.f;
      uint4 kr[EPL], vr[EPL];
      int idx[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        idx[u] = u * SLOTS + g.slot;
        const uint32_t j = (uint32_t)__shfl_sync(0xffffffffu, my_col, idx[u] & 31);
        kr[u] = ldg16(K, j * rq + g.bo);
        vr[u] = ldg16(Vp, j * rv + g.bo);
      }
      float s[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const float full = head_sum<LPH>(P::dot(q, kr[u]));
        s[u] = (idx[u] < n && g.head_ok) ? __fmaf_rn(full, scale_l, b) : M::neg_inf();
      }
      // branchless online update (keeps the V gathers above): a lane with no
      // valid edge so far has m = -inf and ex2(-inf - 0) = 0
      float mx = s[0];
#pragma unroll
      for (int u = 1; u < EPL; ++u) mx = fmaxf(mx, s[u]);
      const float m_new = fmaxf(m, mx);
      const float m_use = (m_new == M::neg_inf()) ? 0.f : m_new;
      const float corr = M::ex(m - m_use);
      l *= corr;
#pragma unroll
      for (int t = 0; t < VW; ++t) acc[t] *= corr;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const float pr = M::ex(s[u] - m_use);
        l += pr;
        const float w = wm ? pr * __ldg(wm + (int64_t)g.hcl * p.E + min(e0 + idx[u], end - 1)) : pr;
        P::axpy(w, vr[u], acc);
      }
      m = m_new;
    }
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1) {
      const float m_o = __shfl_xor_sync(0xffffffffu, m, off);
      const float l_o = __shfl_xor_sync(0xffffffffu, l, off);
      const float m_n = fmaxf(m, m_o);
      const float m_u = (m_n == M::neg_inf()) ? 0.f : m_n;
      const float c_s = M::ex(m - m_u);
      const float c_o = M::ex(m_o - m_u);
      l = l * c_s + l_o * c_o;
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        const float a_o = __shfl_xor_sync(0xffffffffu, acc[t], off);
        acc[t] = acc[t] * c_s + a_o * c_o;
      }
      m = m_n;
    }
    if (g.slot == 0 && g.head_ok) {
#pragma unroll
      for (int t = 0; t < VW; ++t) acc[t] = __fdiv_rn(acc[t], l);
      *reinterpret_cast<uint4*>(O + (uint32_t)i * rv + g.bo) = P::pack(acc);
      if (g.part == 0) LSE[i * p.H + g.hl] = m + M::lg(l);
    }
  }
  int bad = (isnan(chk_q) ? 1 : 0) | (isnan(chk_k) ? 2 : 0) | (isnan(chk_v) ? 4 : 0);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && g.lane == 0) atomicOr(p.err, bad);
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_bwd_rows_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = float(p.scale) * M::kLogScale;
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const char* O = static_cast<const char*>(p.o);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float* __restrict__ LSE = static_cast<const float*>(p.lse);
  float* __restrict__ DELTA = static_cast<float*>(p.delta);
  char* DQ = static_cast<char*>(p.dq);
  float* __restrict__ DB = static_cast<float*>(p.dbias);
  const uint32_t rq = (uint32_t)(p.ldq * sizeof(T)), rv = (uint32_t)(p.ldv * sizeof(T));
  const WarpRange wr = warp_range(p);

  for (int64_t i = wr.first; i < wr.last; i += wr.step) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    float dq[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) dq[t] = 0.f;
    const uint4 d = ldg16(DO, (uint32_t)i * rv + g.bo);
    if (end - beg <= 1) {
      // deg 1: constant weight -> no score gradient (attention.cpp:265-272);
      // delta := dw of the edge so the column pass reproduces ds == 0 exactly
      if (end - beg == 1) {
        const uint4 v = ldg16(Vp, (uint32_t)__ldg(p.cols + beg) * rv + g.bo);
        float dw = head_sum<LPH>(P::dot(d, v));
        if (wm) dw = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + beg), dw);
        if (g.slot == 0 && g.head_ok && g.part == 0) DELTA[i * p.H + g.hl] = dw;
        if (g.lane == 0 && DB) DB[beg] = 0.f;
      }
      if (g.slot == 0 && g.head_ok) *reinterpret_cast<uint4*>(DQ + (uint32_t)i * rq + g.bo) = P::pack(dq);
      continue;
    }
    const uint4 q = ldg16(Q, (uint32_t)i * rq + g.bo);
    const float delta = head_sum<LPH>(P::dot(d, ldg16(O, (uint32_t)i * rv + g.bo)));
    const float lse = __ldg(LSE + i * p.H + g.hcl);
    if (g.slot == 0 && g.head_ok && g.part == 0) DELTA[i * p.H + g.hl] = delta;
    for (int e0 = beg; e0 < end; e0 += CHUNK) {
      const int n = min(CHUNK, end - e0);
      const int my_col = g.lane < n ? __ldg(p.cols + e0 + g.lane) : (int)i;
      const float my_b = (bias && g.lane < n) ? __ldg(bias + e0 + g.lane) * M::kLogScale : 0.f;
      uint4 kr[EPL], vr[EPL];
      int idx[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        idx[u] = u * SLOTS + g.slot;
        const uint32_t j = (uint32_t)__shfl_sync(0xffffffffu, my_col, idx[u] & 31);
        kr[u] = ldg16(K, j * rq + g.bo);
        vr[u] = ldg16(Vp, j * rv + g.bo);
      }
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const float sc = head_sum<LPH>(P::dot(q, kr[u]));
        float dw = head_sum<LPH>(P::dot(d, vr[u]));
        const bool ok = idx[u] < n && g.head_ok;
        const float pr = M::ex(__fmaf_rn(sc, scale_l, b) - lse);
        if (wm) dw = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + min(e0 + idx[u], end - 1)), dw);
        const float ds = ok ? pr * (dw - delta) : 0.f;
        P::axpy(ds, kr[u], dq);
        // dbias_e = sum over heads (parallel.cpp:319): one contribution per head
        float hsum = g.part == 0 ? ds : 0.f;
#pragma unroll
        for (int off = LPH; off < LPN; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
        if (DB && (g.lane % LPN) == 0 && idx[u] < n) DB[e0 + idx[u]] = hsum;
      }
    }
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1)
#pragma unroll
      for (int t = 0; t < VW; ++t) dq[t] += __shfl_xor_sync(0xffffffffu, dq[t], off);
    if (g.slot == 0 && g.head_ok) {
      const float sc = float(p.scale);
#pragma unroll
      for (int t = 0; t < VW; ++t) dq[t] *= sc;
      *reinterpret_cast<uint4*>(DQ + (uint32_t)i * rq + g.bo) = P::pack(dq);
    }
  }
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_bwd_cols_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = float(p.scale) * M::kLogScale;
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float* __restrict__ LSE = static_cast<const float*>(p.lse);
  const float* __restrict__ DELTA = static_cast<const float*>(p.delta);
  char* DK = static_cast<char*>(p.dk_out);
  char* DV = static_cast<char*>(p.dv_out);
  const uint32_t rq = (uint32_t)(p.ldq * sizeof(T)), rv = (uint32_t)(p.ldv * sizeof(T));
  const WarpRange wr = warp_range(p);

  for (int64_t j = wr.first; j < wr.last; j += wr.step) {
    const int beg = __ldg(p.col_ptr + j), end = __ldg(p.col_ptr + j + 1);
    float gk[VW], gv[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) gk[t] = gv[t] = 0.f;
    const uint4 kj = ldg16(K, (uint32_t)j * rq + g.bo);
    const uint4 vj = ldg16(Vp, (uint32_t)j * rv + g.bo);
    for (int e0 = beg; e0 < end; e0 += CHUNK) {
      const int n = min(CHUNK, end - e0);
      const int my_row = g.lane < n ? __ldg(p.csc_row + e0 + g.lane) : (int)j;
      const int my_eid = g.lane < n ? __ldg(p.csc_eid + e0 + g.lane) : 0;
      const float my_b = (bias && g.lane < n) ? __ldg(bias + my_eid) * M::kLogScale : 0.f;
      uint4 qr[EPL], dr[EPL];
      float lse[EPL], dl[EPL];
      int idx[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        idx[u] = u * SLOTS + g.slot;
        const uint32_t i = (uint32_t)__shfl_sync(0xffffffffu, my_row, idx[u] & 31);
        qr[u] = ldg16(Q, i * rq + g.bo);
        dr[u] = ldg16(DO, i * rv + g.bo);
        lse[u] = __ldg(LSE + (int64_t)i * p.H + g.hcl);
        dl[u] = __ldg(DELTA + (int64_t)i * p.H + g.hcl);
      }
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const int e = __shfl_sync(0xffffffffu, my_eid, idx[u] & 31);
        const float sc = head_sum<LPH>(P::dot(qr[u], kj));
        float dw = head_sum<LPH>(P::dot(dr[u], vj));
        const bool ok = idx[u] < n && g.head_ok;
        const float pr = ok ? M::ex(__fmaf_rn(sc, scale_l, b) - lse[u]) : 0.f;
        float pw = pr;
        if (wm) {
          const float mult = __ldg(wm + (int64_t)g.hcl * p.E + e);
          dw = __fmul_rn(mult, dw);
          pw = pr * mult;
        }
        const float ds = ok ? pr * (dw - dl[u]) : 0.f;
        P::axpy(ds, qr[u], gk);
        P::axpy(pw, dr[u], gv);
      }
    }
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1)
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        gk[t] += __shfl_xor_sync(0xffffffffu, gk[t], off);
        gv[t] += __shfl_xor_sync(0xffffffffu, gv[t], off);
      }
    if (g.slot == 0 && g.head_ok) {
      const float sc = float(p.scale);
#pragma unroll
      for (int t = 0; t < VW; ++t) gk[t] *= sc;
      *reinterpret_cast<uint4*>(DK + (uint32_t)j * rq + g.bo) = P::pack(gk);
      *reinterpret_cast<uint4*>(DV + (uint32_t)j * rv + g.bo) = P::pack(gv);
    }
  }
}

}  // namespace gte_b200

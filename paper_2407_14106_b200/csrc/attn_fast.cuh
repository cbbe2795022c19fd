// Memory-level-parallel variant of the sparse graph-attention kernels for the
// aligned shapes that carry the benchmark configs (f32/bf16, head chunks of a
// multiple of 16 bytes, 16-byte aligned rows). Same math, same outputs as the
// generic kernels in attn_sparse.cuh; what changes is the schedule:
//
//   * each lane owns exactly one 16-byte piece of one head of one neighbour
//     (VW = 16/sizeof(T) elements; LPH lanes per head; LPN = pow2(H)*LPH lanes
//     per neighbour; SLOTS = 32/LPN neighbours per warp step),
//   * all K and V (resp. Q and dO) gathers of a chunk of SLOTS*EPL edges are
//     issued back to back as unpredicated 128-bit loads on clamped addresses
//     (invalid slots read the row's own line), so a warp keeps 2*EPL*512 B of
//     gathers in flight instead of one,
//   * the partial dot over VW elements is completed with LPH-1 xor-shuffles,
//   * the vector path is compile-time (no per-load branch).
// Non-finite inputs are detected with x*0 accumulation (NaN iff any operand is
// inf/nan) at one FFMA per element.
#pragma once

#include "attn_sparse.cuh"

namespace gte_b200 {

template <typename T> struct Vec16;
template <> struct Vec16<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void cvt(const uint4& u, float (&o)[4]) {
    o[0] = __uint_as_float(u.x);
    o[1] = __uint_as_float(u.y);
    o[2] = __uint_as_float(u.z);
    o[3] = __uint_as_float(u.w);
  }
  __device__ __forceinline__ static uint4 pack(const float (&o)[4]) {
    return make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]), __float_as_uint(o[3]));
  }
};
template <> struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void cvt(const uint4& u, float (&o)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
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

__device__ __forceinline__ uint4 ldg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int LPH>
__device__ __forceinline__ float head_sum(float x) {
#pragma unroll
  for (int o = 1; o < LPH; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int VW>
__device__ __forceinline__ float dot_vw(const float (&a)[VW], const float (&b)[VW]) {
  float s = __fmul_rn(a[0], b[0]);
#pragma unroll
  for (int t = 1; t < VW; ++t) s = __fmaf_rn(a[t], b[t], s);
  return s;
}

struct FastGeom {
  int lane, slot, hl, part;
  bool head_ok;
  int64_t off;  // element offset of this lane's 16-byte piece inside a row
};

template <int VW, int LPH, int LPN>
__device__ __forceinline__ FastGeom fast_geom(int H, int dh) {
  FastGeom g;
  g.lane = lane_id();
  g.slot = g.lane / LPN;
  const int w = g.lane % LPN;
  g.hl = w / LPH;
  g.part = w % LPH;
  g.head_ok = g.hl < H;
  g.off = g.head_ok ? (int64_t)g.hl * dh + g.part * VW : 0;
  return g;
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_fwd_kernel(SparseArgs p) {
  using V16 = Vec16<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = V16::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<VW, LPH, LPN>(p.H, p.dk);
  const float scale_l = float(p.scale) * M::kLogScale;
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  T* __restrict__ O = static_cast<T*>(p.out);
  float* __restrict__ LSE = static_cast<float*>(p.lse);
  const int64_t rq = p.ldq * (int64_t)sizeof(T), rv = p.ldv * (int64_t)sizeof(T);
  const int64_t bo = g.off * (int64_t)sizeof(T);
  const int hcl = g.head_ok ? g.hl : 0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float chk_q = 0.f, chk_k = 0.f, chk_v = 0.f;

  for (int64_t i = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; i < p.S; i += nwarps) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    float q[VW], acc[VW];
    V16::cvt(ldg16(Q + i * rq + bo), q);
#pragma unroll
    for (int t = 0; t < VW; ++t) {
      acc[t] = 0.f;
      chk_q = __fmaf_rn(q[t], 0.f, chk_q);
    }
    if (end == beg) {
      if (p.forbid_empty && g.lane == 0) atomicMin(p.err + 1, (int)i);
      if (g.slot == 0 && g.head_ok) {
        *reinterpret_cast<uint4*>(O + i * p.ldv + g.off) = V16::pack(acc);
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
        const int j = __shfl_sync(0xffffffffu, my_col, idx[u] & 31);
        kr[u] = ldg16(K + (int64_t)j * rq + bo);
        vr[u] = ldg16(Vp + (int64_t)j * rv + bo);
      }
      float s[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        float kf[VW];
        V16::cvt(kr[u], kf);
        const float part = dot_vw<VW>(q, kf);
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const float full = head_sum<LPH>(part);
        const bool ok = idx[u] < n && g.head_ok;
        if (ok) {
#pragma unroll
          for (int t = 0; t < VW; ++t) chk_k = __fmaf_rn(kf[t], 0.f, chk_k);
        }
        s[u] = ok ? __fmaf_rn(full, scale_l, b) : M::neg_inf();
      }
      // branchless online update (keeps the V gathers hoisted above): a lane
      // with no valid edge so far has m = -inf and ex2(-inf - 0) = 0
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
        const float w = wm ? pr * __ldg(wm + (int64_t)hcl * p.E + min(e0 + idx[u], end - 1)) : pr;
        float vf[VW];
        V16::cvt(vr[u], vf);
        const bool ok = s[u] != M::neg_inf();
#pragma unroll
        for (int t = 0; t < VW; ++t) {
          if (ok) chk_v = __fmaf_rn(vf[t], 0.f, chk_v);
          acc[t] = __fmaf_rn(w, vf[t], acc[t]);
        }
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
      for (int t = 0; t < VW; ++t) acc[t] = acc[t] / l;
      *reinterpret_cast<uint4*>(O + i * p.ldv + g.off) = V16::pack(acc);
      if (g.part == 0) LSE[i * p.H + g.hl] = m + M::lg(l);
    }
  }
  int bad = (g.head_ok && isnan(chk_q) ? 1 : 0) | (isnan(chk_k) ? 2 : 0) | (isnan(chk_v) ? 4 : 0);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && g.lane == 0) atomicOr(p.err, bad);
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_bwd_rows_kernel(SparseArgs p) {
  using V16 = Vec16<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = V16::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<VW, LPH, LPN>(p.H, p.dk);
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
  T* __restrict__ DQ = static_cast<T*>(p.dq);
  float* __restrict__ DB = static_cast<float*>(p.dbias);
  const int64_t rq = p.ldq * (int64_t)sizeof(T), rv = p.ldv * (int64_t)sizeof(T);
  const int64_t bo = g.off * (int64_t)sizeof(T);
  const int hcl = g.head_ok ? g.hl : 0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t i = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; i < p.S; i += nwarps) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    float dq[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) dq[t] = 0.f;
    float d[VW];
    V16::cvt(ldg16(DO + i * rv + bo), d);
    if (end - beg <= 1) {
      // deg 1: constant weight -> no score gradient (attention.cpp:265-272);
      // delta := dw of the edge so the column pass reproduces ds == 0 exactly
      if (end - beg == 1) {
        float vf[VW];
        V16::cvt(ldg16(Vp + (int64_t)__ldg(p.cols + beg) * rv + bo), vf);
        float dw = head_sum<LPH>(dot_vw<VW>(d, vf));
        if (wm && g.head_ok) dw = __fmul_rn(__ldg(wm + (int64_t)g.hl * p.E + beg), dw);
        if (g.slot == 0 && g.head_ok && g.part == 0) DELTA[i * p.H + g.hl] = dw;
        if (g.lane == 0 && DB) DB[beg] = 0.f;
      }
      if (g.slot == 0 && g.head_ok) *reinterpret_cast<uint4*>(DQ + i * p.ldq + g.off) = V16::pack(dq);
      continue;
    }
    float q[VW], o[VW];
    V16::cvt(ldg16(Q + i * rq + bo), q);
    V16::cvt(ldg16(O + i * rv + bo), o);
    const float delta = head_sum<LPH>(dot_vw<VW>(d, o));
    const float lse = g.head_ok ? __ldg(LSE + i * p.H + g.hl) : 0.f;
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
        const int j = __shfl_sync(0xffffffffu, my_col, idx[u] & 31);
        kr[u] = ldg16(K + (int64_t)j * rq + bo);
        vr[u] = ldg16(Vp + (int64_t)j * rv + bo);
      }
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        float kf[VW], vf[VW];
        V16::cvt(kr[u], kf);
        V16::cvt(vr[u], vf);
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const float sc = head_sum<LPH>(dot_vw<VW>(q, kf));
        float dw = head_sum<LPH>(dot_vw<VW>(d, vf));
        const bool ok = idx[u] < n && g.head_ok;
        const float s = __fmaf_rn(sc, scale_l, b);
        const float pr = M::ex(s - lse);
        if (wm) dw = __fmul_rn(__ldg(wm + (int64_t)hcl * p.E + min(e0 + idx[u], end - 1)), dw);
        const float ds = ok ? pr * (dw - delta) : 0.f;
#pragma unroll
        for (int t = 0; t < VW; ++t) dq[t] = __fmaf_rn(ds, kf[t], dq[t]);
        // dbias_e = sum over heads (parallel.cpp:319): one contribution per head
        float hsum = g.part == 0 ? ds : 0.f;
#pragma unroll
        for (int off = 1; off < LPN; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
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
      *reinterpret_cast<uint4*>(DQ + i * p.ldq + g.off) = V16::pack(dq);
    }
  }
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) fast_bwd_cols_kernel(SparseArgs p) {
  using V16 = Vec16<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = V16::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int CHUNK = SLOTS * EPL;
  const FastGeom g = fast_geom<VW, LPH, LPN>(p.H, p.dk);
  const float scale_l = float(p.scale) * M::kLogScale;
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float* __restrict__ LSE = static_cast<const float*>(p.lse);
  const float* __restrict__ DELTA = static_cast<const float*>(p.delta);
  T* __restrict__ DK = static_cast<T*>(p.dk_out);
  T* __restrict__ DV = static_cast<T*>(p.dv_out);
  const int64_t rq = p.ldq * (int64_t)sizeof(T), rv = p.ldv * (int64_t)sizeof(T);
  const int64_t bo = g.off * (int64_t)sizeof(T);
  const int hcl = g.head_ok ? g.hl : 0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t j = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; j < p.S; j += nwarps) {
    const int beg = __ldg(p.col_ptr + j), end = __ldg(p.col_ptr + j + 1);
    float gk[VW], gv[VW], kf[VW], vf[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) gk[t] = gv[t] = 0.f;
    V16::cvt(ldg16(K + j * rq + bo), kf);
    V16::cvt(ldg16(Vp + j * rv + bo), vf);
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
        const int i = __shfl_sync(0xffffffffu, my_row, idx[u] & 31);
        qr[u] = ldg16(Q + (int64_t)i * rq + bo);
        dr[u] = ldg16(DO + (int64_t)i * rv + bo);
        lse[u] = __ldg(LSE + (int64_t)i * p.H + hcl);
        dl[u] = __ldg(DELTA + (int64_t)i * p.H + hcl);
      }
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        float qf[VW], df[VW];
        V16::cvt(qr[u], qf);
        V16::cvt(dr[u], df);
        const float b = __shfl_sync(0xffffffffu, my_b, idx[u] & 31);
        const int e = __shfl_sync(0xffffffffu, my_eid, idx[u] & 31);
        const float sc = head_sum<LPH>(dot_vw<VW>(qf, kf));
        float dw = head_sum<LPH>(dot_vw<VW>(df, vf));
        const bool ok = idx[u] < n && g.head_ok;
        const float s = __fmaf_rn(sc, scale_l, b);
        const float pr = ok ? M::ex(s - lse[u]) : 0.f;
        float pw = pr;
        if (wm) {
          const float mult = __ldg(wm + (int64_t)hcl * p.E + e);
          dw = __fmul_rn(mult, dw);
          pw = pr * mult;
        }
        const float ds = ok ? pr * (dw - dl[u]) : 0.f;
#pragma unroll
        for (int t = 0; t < VW; ++t) {
          gk[t] = __fmaf_rn(ds, qf[t], gk[t]);
          gv[t] = __fmaf_rn(pw, df[t], gv[t]);
        }
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
      *reinterpret_cast<uint4*>(DK + j * p.ldq + g.off) = V16::pack(gk);
      *reinterpret_cast<uint4*>(DV + j * p.ldv + g.off) = V16::pack(gv);
    }
  }
}

}  // namespace gte_b200

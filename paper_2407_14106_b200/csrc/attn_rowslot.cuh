// "Row-slot" schedule for the sparse graph-attention kernels (aligned f32/bf16
// shapes). ncu on the one-warp-per-row kernels showed ~50 warp-instructions
// per edge and long-scoreboard stalls on the row_ptr -> cols -> K/V dependency
// chain of every row, with a per-row cross-slot softmax merge on top. Here a
// warp runs SLOTS = 32/LPN rows at once, one per slot of LPN lanes (a lane =
// one 16-byte piece of one head):
//
//   * each slot streams its own row EPL edges per step, keeping its own online
//     softmax state — no cross-slot merge, no padding of short rows to a
//     32-edge chunk;
//   * when a slot's row ends it is finalised (predicated stores) and the slot
//     takes the next row of the CTA's contiguous range from a shared-memory
//     counter (warp-aggregated atomics), so hub rows do not stall the warp;
//   * the K/V gathers of a step are issued together, before any use.
// Math, numerics and outputs are identical to attn_fast.cuh (same Piece dot /
// axpy helpers, same log2-domain softmax, same degree-1 exactness).
#pragma once

#include "attn_fast.cuh"

namespace gte_b200 {

// Per-warp row assignment from the CTA range [r0, r1): slot s of warp w starts
// at r0 + w*SLOTS + s; finished slots draw the next rows in slot order.
template <int SLOTS, int LPN>
struct RowQueue {
  int* next;  // shared
  int r1;
  __device__ __forceinline__ int refill(bool need, int lane) {
    const unsigned leaders = __ballot_sync(0xffffffffu, need && (lane % LPN) == 0);
    const int cnt = __popc(leaders);
    int base = 0;
    if (cnt) {
      if (lane == 0) base = atomicAdd(next, cnt);
      base = __shfl_sync(0xffffffffu, base, 0);
    }
    const int slot_leader = (lane / LPN) * LPN;
    const int rank = __popc(leaders & ((1u << slot_leader) - 1u));
    const int row = base + rank;
    return (need && row < r1) ? row : -1;
  }
};

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) slot_fwd_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  __shared__ int s_next;
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
  const int r0 = (int)((int64_t)blockIdx.x * p.rows_per_cta);
  const int r1 = (int)min((int64_t)r0 + p.rows_per_cta, p.S);
  const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) s_next = r0 + nwarp * SLOTS;
  __syncthreads();
  RowQueue<SLOTS, LPN> rq_{&s_next, r1};

  float chk_q = 0.f, chk_k = 0.f, chk_v = 0.f;
  int i = r0 + warp * SLOTS + g.slot;
  if (i >= r1) i = -1;
  int e = 0, end = 0, beg = 0;
  uint4 q = make_uint4(0, 0, 0, 0);
  float m = M::neg_inf(), l = 0.f, acc[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) acc[t] = 0.f;
  auto start_row = [&](int row) {
    if (row >= 0) {
      beg = e = __ldg(p.row_ptr + row);
      end = __ldg(p.row_ptr + row + 1);
      q = ldg16(Q, (uint32_t)row * rq + g.bo);
      if (g.head_ok) {  // own-row finiteness (attention.cpp:20-22)
        chk_q = P::finite_probe(q, chk_q);
        chk_k = P::finite_probe(ldg16(K, (uint32_t)row * rq + g.bo), chk_k);
        chk_v = P::finite_probe(ldg16(Vp, (uint32_t)row * rv + g.bo), chk_v);
      }
    } else {
      beg = e = end = 0;
    }
    m = M::neg_inf();
    l = 0.f;
#pragma unroll
    for (int t = 0; t < VW; ++t) acc[t] = 0.f;
  };
  start_row(i);

  while (__any_sync(0xffffffffu, i >= 0)) {
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
    bool ok[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int eu = e + u;
      ok[u] = i >= 0 && eu < end;
      const uint32_t j = ok[u] ? (uint32_t)__ldg(p.cols + eu) : (uint32_t)max(i, 0);
      bl[u] = (bias && ok[u]) ? __ldg(bias + eu) : 0.f;
      kr[u] = ldg16(K, j * rq + g.bo);
      vr[u] = ldg16(Vp, j * rv + g.bo);
    }
    float s[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float full = head_sum<LPH>(P::dot(q, kr[u]));
      s[u] = (ok[u] && g.head_ok) ? __fmaf_rn(full, scale_l, bl[u] * M::kLogScale) : M::neg_inf();
    }
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
      const float w = (wm && ok[u]) ? pr * __ldg(wm + (int64_t)g.hcl * p.E + e + u) : pr;
      P::axpy(w, vr[u], acc);
    }
    m = m_new;
    e += EPL;
    const bool done = i >= 0 && e >= end;
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
        if (end == beg) {  // empty row: zero output (attention.cpp:119-125)
          if (p.forbid_empty && (g.lane % LPN) == 0) atomicMin(p.err + 1, i);
          if (g.head_ok) {
            *reinterpret_cast<uint4*>(O + (uint32_t)i * rv + g.bo) = P::pack(acc);
            if (g.part == 0) LSE[(int64_t)i * p.H + g.hl] = M::neg_inf();
          }
        } else if (g.head_ok) {
          const float inv = __frcp_rn(l);  // l == 1 (degree-1 rows) stays exact
#pragma unroll
          for (int t = 0; t < VW; ++t) acc[t] *= inv;
          *reinterpret_cast<uint4*>(O + (uint32_t)i * rv + g.bo) = P::pack(acc);
          if (g.part == 0) LSE[(int64_t)i * p.H + g.hl] = m + M::lg(l);
        }
      }
      const int nrow = rq_.refill(done, g.lane);
      if (done) {
        i = nrow;
        start_row(i);
      }
    }
  }
  int bad = (isnan(chk_q) ? 1 : 0) | (isnan(chk_k) ? 2 : 0) | (isnan(chk_v) ? 4 : 0);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && g.lane == 0) atomicOr(p.err, bad);
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) slot_bwd_rows_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  __shared__ int s_next;
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
  const int r0 = (int)((int64_t)blockIdx.x * p.rows_per_cta);
  const int r1 = (int)min((int64_t)r0 + p.rows_per_cta, p.S);
  const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) s_next = r0 + nwarp * SLOTS;
  __syncthreads();
  RowQueue<SLOTS, LPN> rq_{&s_next, r1};

  int i = r0 + warp * SLOTS + g.slot;
  if (i >= r1) i = -1;
  int e = 0, end = 0, beg = 0;
  uint4 q = make_uint4(0, 0, 0, 0), d = q;
  float lse = 0.f, delta = 0.f, dq[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) dq[t] = 0.f;
  // Warp-wide (it shuffles); only lanes with `take` adopt the new row.
  auto load_row = [&](int row, bool take) {
    const int rc = row >= 0 ? row : 0;
    const int b0 = __ldg(p.row_ptr + rc), b1 = __ldg(p.row_ptr + rc + 1);
    const uint4 q_ = ldg16(Q, (uint32_t)rc * rq + g.bo);
    const uint4 d_ = ldg16(DO, (uint32_t)rc * rv + g.bo);
    const float lse_ = __ldg(LSE + (int64_t)rc * p.H + g.hcl);
    const bool single = b1 - b0 == 1;
    const uint32_t js = (b1 > b0) ? (uint32_t)__ldg(p.cols + b0) : (uint32_t)rc;
    // deg 1: constant weight -> no score gradient (attention.cpp:265-272);
    // delta := dw of the edge so the column pass reproduces ds == 0 exactly
    float dw1 = head_sum<LPH>(P::dot(d_, ldg16(Vp, js * rv + g.bo)));
    if (wm && single) dw1 = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + b0), dw1);
    const float dd = head_sum<LPH>(P::dot(d_, ldg16(O, (uint32_t)rc * rv + g.bo)));
    if (take) {
#pragma unroll
      for (int t = 0; t < VW; ++t) dq[t] = 0.f;
      if (row >= 0) {
        beg = e = b0;
        end = b1;
        q = q_;
        d = d_;
        lse = lse_;
        delta = single ? dw1 : dd;
        if (g.head_ok && g.part == 0) DELTA[(int64_t)row * p.H + g.hl] = delta;
      } else {
        beg = e = end = 0;
      }
    }
  };
  load_row(i, true);

  while (__any_sync(0xffffffffu, i >= 0)) {
    const bool single = end - beg == 1;
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
    bool ok[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int eu = e + u;
      ok[u] = i >= 0 && eu < end;
      const uint32_t j = ok[u] ? (uint32_t)__ldg(p.cols + eu) : (uint32_t)max(i, 0);
      bl[u] = (bias && ok[u]) ? __ldg(bias + eu) : 0.f;
      kr[u] = ldg16(K, j * rq + g.bo);
      vr[u] = ldg16(Vp, j * rv + g.bo);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(q, kr[u]));
      float dw = head_sum<LPH>(P::dot(d, vr[u]));
      const float pr = M::ex(__fmaf_rn(sc, scale_l, bl[u] * M::kLogScale) - lse);
      if (wm && ok[u]) dw = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + e + u), dw);
      const float ds = (ok[u] && g.head_ok && !single) ? pr * (dw - delta) : 0.f;
      P::axpy(ds, kr[u], dq);
      // dbias_e = sum over heads (parallel.cpp:319): one contribution per head
      float hsum = g.part == 0 ? ds : 0.f;
#pragma unroll
      for (int off = LPH; off < LPN; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
      if (DB && ok[u] && (g.lane % LPN) == 0) DB[e + u] = hsum;
    }
    e += EPL;
    const bool done = i >= 0 && e >= end;
    if (__any_sync(0xffffffffu, done)) {
      if (done && g.head_ok) {
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < VW; ++t) dq[t] *= sc;
        *reinterpret_cast<uint4*>(DQ + (uint32_t)i * rq + g.bo) = P::pack(dq);
      }
      const int nrow = rq_.refill(done, g.lane);
      if (done) i = nrow;
      load_row(done ? i : -1, done);
    }
  }
}

// ---------------------------------------------------------------------------
template <typename T, int LPH, int LPN, int EPL>
__global__ void __launch_bounds__(256) slot_bwd_cols_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  __shared__ int s_next;
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
  const int r0 = (int)((int64_t)blockIdx.x * p.rows_per_cta);
  const int r1 = (int)min((int64_t)r0 + p.rows_per_cta, p.S);
  const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) s_next = r0 + nwarp * SLOTS;
  __syncthreads();
  RowQueue<SLOTS, LPN> rq_{&s_next, r1};

  int j = r0 + warp * SLOTS + g.slot;
  if (j >= r1) j = -1;
  int e = 0, end = 0;
  uint4 kj = make_uint4(0, 0, 0, 0), vj = kj;
  float gk[VW], gv[VW];
  auto start_col = [&](int col) {
#pragma unroll
    for (int t = 0; t < VW; ++t) gk[t] = gv[t] = 0.f;
    if (col < 0) {
      e = end = 0;
      return;
    }
    e = __ldg(p.col_ptr + col);
    end = __ldg(p.col_ptr + col + 1);
    kj = ldg16(K, (uint32_t)col * rq + g.bo);
    vj = ldg16(Vp, (uint32_t)col * rv + g.bo);
  };
  start_col(j);

  while (__any_sync(0xffffffffu, j >= 0)) {
    uint4 qr[EPL], dr[EPL];
    float lse[EPL], dl[EPL], bl[EPL], mult[EPL];
    bool ok[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int eu = e + u;
      ok[u] = j >= 0 && eu < end;
      const uint32_t i = ok[u] ? (uint32_t)__ldg(p.csc_row + eu) : (uint32_t)max(j, 0);
      const int eid = ok[u] ? __ldg(p.csc_eid + eu) : 0;
      qr[u] = ldg16(Q, i * rq + g.bo);
      dr[u] = ldg16(DO, i * rv + g.bo);
      lse[u] = __ldg(LSE + (int64_t)i * p.H + g.hcl);
      dl[u] = __ldg(DELTA + (int64_t)i * p.H + g.hcl);
      bl[u] = (bias && ok[u]) ? __ldg(bias + eid) : 0.f;
      mult[u] = (wm && ok[u]) ? __ldg(wm + (int64_t)g.hcl * p.E + eid) : 1.f;
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(qr[u], kj));
      float dw = head_sum<LPH>(P::dot(dr[u], vj));
      const bool v_ok = ok[u] && g.head_ok;
      const float pr = v_ok ? M::ex(__fmaf_rn(sc, scale_l, bl[u] * M::kLogScale) - lse[u]) : 0.f;
      float pw = pr;
      if (wm) {
        dw = __fmul_rn(mult[u], dw);
        pw = pr * mult[u];
      }
      const float ds = v_ok ? pr * (dw - dl[u]) : 0.f;
      P::axpy(ds, qr[u], gk);
      P::axpy(pw, dr[u], gv);
    }
    e += EPL;
    const bool done = j >= 0 && e >= end;
    if (__any_sync(0xffffffffu, done)) {
      if (done && g.head_ok) {
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < VW; ++t) gk[t] *= sc;
        *reinterpret_cast<uint4*>(DK + (uint32_t)j * rq + g.bo) = P::pack(gk);
        *reinterpret_cast<uint4*>(DV + (uint32_t)j * rv + g.bo) = P::pack(gv);
      }
      const int ncol = rq_.refill(done, g.lane);
      if (done) {
        j = ncol;
        start_col(j);
      }
    }
  }
}

}  // namespace gte_b200

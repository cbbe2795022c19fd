// Topology-induced sparse graph attention, forward + atomic-free backward,
// hand-written for sm_100a.
//
// Replaces the reference's per-head scalar loops:
//   forward   proj/src/attention.cpp:96-162   (sparse_attention)
//   backward  proj/src/attention.cpp:241-320  (sparse_attention_backward)
// and, when H > 1, the per-head loop + dbias head sum of the distributed layer
//   proj/src/parallel.cpp:234-247, :307-323.
//
// Layout: Q/K [S x ldq], V/O/dO [S x ldv]; head h owns columns [h*dk, (h+1)*dk)
// (resp. dv) — the reference's multi-head layout (parallel.cpp:236-238).
// Pattern: int32 CSR (row_ptr, cols), plus a CSC view (col_ptr, csc_row,
// csc_eid) built once per pattern for the backward's key/value pass.
//
// Warp mapping (one warp per row / per column): lane = slot * LPN + head, where
// LPN = next_pow2(H) lanes cover all heads of one neighbour and the warp keeps
// SLOTS = 32 / LPN neighbours in flight; each lane holds its head's q/acc
// (<= DHT elements) in registers and gathers the neighbour's K/V head chunk
// with 16-byte loads. Scores live in registers; softmax is online per chunk of
// SLOTS*EPL edges and merged across slots with shuffles at the end of the row.
//
// Backward is two passes, no atomics:
//   A (rows, CSR): delta_i = dO_i.O_i, recompute p, ds; dQ_i, dbias_e (sum over
//                  heads via shuffles).
//   B (cols, CSC): recompute p, ds per in-edge; dK_j, dV_j.
#pragma once

#include "common.cuh"

namespace gte_b200 {

struct SparseArgs {
  int64_t S = 0, E = 0;
  int H = 1, dk = 1, dv = 1;
  int64_t ldq = 1, ldv = 1;
  const int32_t* row_ptr = nullptr;
  const int32_t* cols = nullptr;
  const int32_t* col_ptr = nullptr;
  const int32_t* csc_row = nullptr;
  const int32_t* csc_eid = nullptr;
  const void* q = nullptr;
  const void* k = nullptr;
  const void* v = nullptr;
  const void* o = nullptr;
  const void* dout = nullptr;
  const void* bias = nullptr;   // A[E] or null (shared by heads)
  const void* wmult = nullptr;  // A[H*E] head-major or null
  void* out = nullptr;
  void* lse = nullptr;    // A[S*H]
  void* delta = nullptr;  // A[S*H]
  void* dq = nullptr;
  void* dk_out = nullptr;
  void* dv_out = nullptr;
  void* dbias = nullptr;  // A[E]
  double scale = 1.0;
  // tile kernels: float(scale) * log2(e) and the row strides in bytes,
  // computed once on the host (fill_common) so the kernels' main loops read
  // them as uniform operands instead of rebuilding them every step
  float scale_l = 0.f;
  uint32_t rq_bytes = 0, rv_bytes = 0;
  int forbid_empty = 0;
  int vec_qk = 0, vec_v = 0;
  int* err = nullptr;  // [0] non-finite flag, [1] first empty row (atomicMin)
  // Each CTA owns a contiguous range of rows (columns for the CSC pass); its
  // warps stride through it. Contiguous ranges keep a cluster-ordered
  // sequence's neighbour rows hot in that SM's L1.
  int64_t rows_per_cta = 8;
  // tile kernels (attn_tile.cuh): execution plan of the CSR pass (order of
  // the non-hub rows, tile boundaries into it, hub rows) and of the CSC pass
  // (same over columns), and the packed (lse, delta) workspace [S x H] float2
  // written by the CSR pass for the CSC pass.
  const int32_t* order = nullptr;
  const int32_t* tiles = nullptr;
  const int32_t* hubs = nullptr;
  const int32_t* order_c = nullptr;
  const int32_t* tiles_c = nullptr;
  const int32_t* hubs_c = nullptr;
  int n_tiles = 0, n_hubs = 0, n_tiles_c = 0, n_hubs_c = 0;
  void* lsedelta = nullptr;
  // ECR split (ecr_tile.cuh): the pattern here is the remainder of a layout
  // whose dense sub-blocks ran on the tensor pipe. eid maps a CSR position to
  // the original edge id (bias / weight_mult / dbias slots; the CSC view's
  // csc_eid is already original). Per row (column) the tile partials to fold
  // in are [inc_ptr[i], inc_ptr[i+1]) ([cinc_ptr[j], cinc_ptr[j+1])), rows of
  // part_d floats: forward (m, l) in part_ml + unnormalised acc in part_acc;
  // backward dQ in part_acc, dK / dV in part_dk / part_dv.
  const int32_t* eid = nullptr;
  const int32_t* inc_ptr = nullptr;
  const int32_t* cinc_ptr = nullptr;
  const float2* part_ml = nullptr;
  const float* part_acc = nullptr;
  const float* part_dk = nullptr;
  const float* part_dv = nullptr;
  int part_d = 0;
};

struct WarpRange {
  int64_t first, last, step;
};

__device__ __forceinline__ WarpRange warp_range(const SparseArgs& p) {
  const int64_t r0 = (int64_t)blockIdx.x * p.rows_per_cta;
  const int64_t r1 = r0 + p.rows_per_cta < p.S ? r0 + p.rows_per_cta : p.S;
  return {r0 + (threadIdx.x >> 5), r1, (int64_t)(blockDim.x >> 5)};
}

// Edges per lane per chunk: up to LPN (one full warp of neighbours per chunk),
// at most 8, and bounded so the unrolled gathers keep <= budget/DHT rows live.
__host__ __device__ constexpr int epl_for(int lpn, int dht, int budget) {
  int e = lpn < 8 ? lpn : 8;
  int cap = budget / dht;
  if (cap < 1) cap = 1;
  return e < cap ? e : cap;
}

template <typename A>
__device__ __forceinline__ bool finite_acc(A x) {
  return isfinite(x);
}

// score in the kernel's softmax domain: (q.k) * scale (+ bias), x log2e for fp32
template <typename A, int DHT>
__device__ __forceinline__ A score_of(const A (&q)[DHT], const A (&k)[DHT], A scale_l, A b_l) {
  using M = SoftmaxMath<A>;
  return M::fma(dot_chunk<A, DHT>(q, k), scale_l, b_l);
}

// ----------------------------------------------------------------------------
// forward
// ----------------------------------------------------------------------------
// chunks per partial of the backward's two-level sums; on for head chunks
// up to 32 elements (DHT = 64 already spills: it keeps one running sum)
constexpr int kSumBlock = 64;
__host__ __device__ constexpr bool two_level_sums(int dht) { return dht <= 32; }

template <typename T, int DHT, int LPN>
__global__ void __launch_bounds__(256) sparse_fwd_kernel(SparseArgs p) {
  using A = typename AccOf<T>::type;
  using M = SoftmaxMath<A>;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int EPL = epl_for(LPN, DHT, 128 / (int)sizeof(A) * 4);
  constexpr int CHUNK = SLOTS * EPL;
  const int lane = lane_id(), slot = lane / LPN, hl = lane % LPN;
  const bool head_ok = hl < p.H;
  const A scale_l = A(p.scale) * A(M::kLogScale);
  const T* __restrict__ Q = static_cast<const T*>(p.q);
  const T* __restrict__ K = static_cast<const T*>(p.k);
  const T* __restrict__ V = static_cast<const T*>(p.v);
  const A* __restrict__ bias = static_cast<const A*>(p.bias);
  const A* __restrict__ wm = static_cast<const A*>(p.wmult);
  T* __restrict__ O = static_cast<T*>(p.out);
  A* __restrict__ LSE = static_cast<A*>(p.lse);
  const bool vqk = p.vec_qk, vv = p.vec_v;
  const int64_t qoff = (int64_t)hl * p.dk, voff = (int64_t)hl * p.dv;
  const WarpRange wr = warp_range(p);
  int bad = 0;  // bit 0: Q, bit 1: K, bit 2: V non-finite

  for (int64_t i = wr.first; i < wr.last; i += wr.step) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    A q[DHT], acc[DHT];
#pragma unroll
    for (int t = 0; t < DHT; ++t) acc[t] = A(0);
    if (head_ok) {
      load_chunk<T, DHT>(Q + i * p.ldq + qoff, p.dk, vqk, q);
#pragma unroll
      for (int t = 0; t < DHT; ++t) bad |= finite_acc(q[t]) ? 0 : 1;
    } else {
#pragma unroll
      for (int t = 0; t < DHT; ++t) q[t] = A(0);
    }
    if (end == beg) {
      if (p.forbid_empty && lane == 0) atomicMin(p.err + 1, (int)i);
      if (slot == 0 && head_ok) {
        store_chunk<T, DHT>(O + i * p.ldv + voff, p.dv, vv, acc);
        LSE[i * p.H + hl] = M::neg_inf();
      }
      continue;
    }
    A m = M::neg_inf(), l = A(0);
    for (int e0 = beg; e0 < end; e0 += CHUNK) {
      const int n = min(CHUNK, end - e0);
      const int my_col = lane < n ? __ldg(p.cols + e0 + lane) : 0;
      const A my_b = (bias && lane < n) ? __ldg(bias + e0 + lane) * A(M::kLogScale) : A(0);
      A s[EPL];
      int jj[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int idx = u * SLOTS + slot;
        jj[u] = __shfl_sync(0xffffffffu, my_col, idx & 31);
        const A b = __shfl_sync(0xffffffffu, my_b, idx & 31);
        s[u] = M::neg_inf();
        if (idx < n && head_ok) {
          A kr[DHT];
          load_chunk<T, DHT>(K + (int64_t)jj[u] * p.ldq + qoff, p.dk, vqk, kr);
#pragma unroll
          for (int t = 0; t < DHT; ++t) bad |= finite_acc(kr[t]) ? 0 : 2;
          s[u] = score_of<A, DHT>(q, kr, scale_l, b);
        }
      }
      A mx = s[0];
#pragma unroll
      for (int u = 1; u < EPL; ++u) mx = mx > s[u] ? mx : s[u];
      if (mx != M::neg_inf()) {  // else: this lane saw no edge in the chunk
        const A m_new = m > mx ? m : mx;
        const A corr = (m == M::neg_inf()) ? A(0) : M::ex(m - m_new);
        l *= corr;
#pragma unroll
        for (int t = 0; t < DHT; ++t) acc[t] *= corr;
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const int idx = u * SLOTS + slot;
          if (idx < n && head_ok) {
            const A pr = M::ex(s[u] - m_new);
            l += pr;
            const A w = wm ? pr * __ldg(wm + (int64_t)hl * p.E + e0 + idx) : pr;
            A vr[DHT];
            load_chunk<T, DHT>(V + (int64_t)jj[u] * p.ldv + voff, p.dv, vv, vr);
#pragma unroll
            for (int t = 0; t < DHT; ++t) {
              bad |= finite_acc(vr[t]) ? 0 : 4;
              acc[t] = M::fma(w, vr[t], acc[t]);
            }
          }
        }
        m = m_new;
      }
    }
    // merge the SLOTS partial softmax states
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1) {
      const A m_o = __shfl_xor_sync(0xffffffffu, m, off);
      const A l_o = __shfl_xor_sync(0xffffffffu, l, off);
      const A m_n = m > m_o ? m : m_o;
      const A c_s = (m == M::neg_inf()) ? A(0) : M::ex(m - m_n);
      const A c_o = (m_o == M::neg_inf()) ? A(0) : M::ex(m_o - m_n);
      l = l * c_s + l_o * c_o;
#pragma unroll
      for (int t = 0; t < DHT; ++t) {
        const A a_o = __shfl_xor_sync(0xffffffffu, acc[t], off);
        acc[t] = acc[t] * c_s + a_o * c_o;
      }
      m = m_n;
    }
    if (slot == 0 && head_ok) {
#pragma unroll
      for (int t = 0; t < DHT; ++t) acc[t] = acc[t] / l;
      store_chunk<T, DHT>(O + i * p.ldv + voff, p.dv, vv, acc);
      LSE[i * p.H + hl] = m + M::lg(l);
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(p.err, bad);
}

// ----------------------------------------------------------------------------
// backward pass A: rows (CSR)
// ----------------------------------------------------------------------------
template <typename T, int DHT, int LPN>
__global__ void __launch_bounds__(256) sparse_bwd_rows_kernel(SparseArgs p) {
  using A = typename AccOf<T>::type;
  using M = SoftmaxMath<A>;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int EPL = epl_for(LPN, DHT, 64 / (int)sizeof(A) * 4);
  constexpr int CHUNK = SLOTS * EPL;
  const int lane = lane_id(), slot = lane / LPN, hl = lane % LPN;
  const bool head_ok = hl < p.H;
  const A scale_l = A(p.scale) * A(M::kLogScale);
  const T* __restrict__ Q = static_cast<const T*>(p.q);
  const T* __restrict__ K = static_cast<const T*>(p.k);
  const T* __restrict__ V = static_cast<const T*>(p.v);
  const T* __restrict__ O = static_cast<const T*>(p.o);
  const T* __restrict__ DO = static_cast<const T*>(p.dout);
  const A* __restrict__ bias = static_cast<const A*>(p.bias);
  const A* __restrict__ wm = static_cast<const A*>(p.wmult);
  const A* __restrict__ LSE = static_cast<const A*>(p.lse);
  A* __restrict__ DELTA = static_cast<A*>(p.delta);
  T* __restrict__ DQ = static_cast<T*>(p.dq);
  A* __restrict__ DB = static_cast<A*>(p.dbias);
  const bool vqk = p.vec_qk, vv = p.vec_v;
  const int64_t qoff = (int64_t)hl * p.dk, voff = (int64_t)hl * p.dv;
  const WarpRange wr = warp_range(p);

  for (int64_t i = wr.first; i < wr.last; i += wr.step) {
    const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
    A dq[DHT];
#pragma unroll
    for (int t = 0; t < DHT; ++t) dq[t] = A(0);
    if (end - beg <= 1) {
      // deg 0: nothing. deg 1: constant weight, no score gradient
      // (attention.cpp:265-272); delta is set to the single edge's dw so that
      // pass B reproduces ds == 0 exactly.
      if (end - beg == 1 && head_ok) {
        A d[DHT], vr[DHT];
        load_chunk<T, DHT>(DO + i * p.ldv + voff, p.dv, vv, d);
        const int j = __ldg(p.cols + beg);
        load_chunk<T, DHT>(V + (int64_t)j * p.ldv + voff, p.dv, vv, vr);
        A dw = dot_chunk<A, DHT>(d, vr);
        if (wm) dw = M::mul(__ldg(wm + (int64_t)hl * p.E + beg), dw);
        if (slot == 0) DELTA[i * p.H + hl] = dw;
      }
      if (end - beg == 1 && lane == 0 && DB) DB[beg] = A(0);
      if (slot == 0 && head_ok) store_chunk<T, DHT>(DQ + i * p.ldq + qoff, p.dk, vqk, dq);
      continue;
    }
    A q[DHT], d[DHT], lse = A(0), delta = A(0);
    if (head_ok) {
      A o[DHT];
      load_chunk<T, DHT>(Q + i * p.ldq + qoff, p.dk, vqk, q);
      load_chunk<T, DHT>(DO + i * p.ldv + voff, p.dv, vv, d);
      load_chunk<T, DHT>(O + i * p.ldv + voff, p.dv, vv, o);
      delta = dot_chunk<A, DHT>(d, o);
      lse = __ldg(LSE + i * p.H + hl);
      if (slot == 0) DELTA[i * p.H + hl] = delta;
    } else {
#pragma unroll
      for (int t = 0; t < DHT; ++t) q[t] = d[t] = A(0);
    }
    A tq[DHT];  // two-level sum as in the CSC pass (degree-S hub rows)
#pragma unroll
    for (int t = 0; t < DHT; ++t) tq[t] = A(0);
    for (int b0 = beg; b0 < end; b0 += kSumBlock * CHUNK) {
    const int b1 = min(end, b0 + kSumBlock * CHUNK);
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) dq[t] = A(0);
    for (int e0 = b0; e0 < b1; e0 += CHUNK) {
      const int n = min(CHUNK, b1 - e0);
      const int my_col = lane < n ? __ldg(p.cols + e0 + lane) : 0;
      const A my_b = (bias && lane < n) ? __ldg(bias + e0 + lane) * A(M::kLogScale) : A(0);
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int idx = u * SLOTS + slot;
        const int j = __shfl_sync(0xffffffffu, my_col, idx & 31);
        const A b = __shfl_sync(0xffffffffu, my_b, idx & 31);
        A ds = A(0);
        if (idx < n && head_ok) {
          A kr[DHT], vr[DHT];
          load_chunk<T, DHT>(K + (int64_t)j * p.ldq + qoff, p.dk, vqk, kr);
          load_chunk<T, DHT>(V + (int64_t)j * p.ldv + voff, p.dv, vv, vr);
          const A s = score_of<A, DHT>(q, kr, scale_l, b);
          const A pr = M::ex(s - lse);
          A dw = dot_chunk<A, DHT>(d, vr);
          if (wm) dw = M::mul(__ldg(wm + (int64_t)hl * p.E + e0 + idx), dw);
          ds = pr * (dw - delta);
#pragma unroll
          for (int t = 0; t < DHT; ++t) dq[t] = M::fma(ds, kr[t], dq[t]);
        }
        // dbias_e = sum over heads of ds (parallel.cpp:319)
#pragma unroll
        for (int off = 1; off < LPN; off <<= 1) ds += __shfl_xor_sync(0xffffffffu, ds, off);
        if (DB && hl == 0 && idx < n) DB[e0 + idx] = ds;
      }
    }
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) tq[t] += dq[t];
    }
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) dq[t] = tq[t];
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1)
#pragma unroll
      for (int t = 0; t < DHT; ++t) dq[t] += __shfl_xor_sync(0xffffffffu, dq[t], off);
    if (slot == 0 && head_ok) {
      const A sc = A(p.scale);
#pragma unroll
      for (int t = 0; t < DHT; ++t) dq[t] *= sc;
      store_chunk<T, DHT>(DQ + i * p.ldq + qoff, p.dk, vqk, dq);
    }
  }
}

// ----------------------------------------------------------------------------
// backward pass B: columns (CSC) -> dK, dV
// ----------------------------------------------------------------------------
template <typename T, int DHT, int LPN>
__global__ void __launch_bounds__(256) sparse_bwd_cols_kernel(SparseArgs p) {
  using A = typename AccOf<T>::type;
  using M = SoftmaxMath<A>;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int EPL = epl_for(LPN, DHT, 64 / (int)sizeof(A) * 4);
  constexpr int CHUNK = SLOTS * EPL;
  const int lane = lane_id(), slot = lane / LPN, hl = lane % LPN;
  const bool head_ok = hl < p.H;
  const A scale_l = A(p.scale) * A(M::kLogScale);
  const T* __restrict__ Q = static_cast<const T*>(p.q);
  const T* __restrict__ K = static_cast<const T*>(p.k);
  const T* __restrict__ V = static_cast<const T*>(p.v);
  const T* __restrict__ DO = static_cast<const T*>(p.dout);
  const A* __restrict__ bias = static_cast<const A*>(p.bias);
  const A* __restrict__ wm = static_cast<const A*>(p.wmult);
  const A* __restrict__ LSE = static_cast<const A*>(p.lse);
  const A* __restrict__ DELTA = static_cast<const A*>(p.delta);
  T* __restrict__ DK = static_cast<T*>(p.dk_out);
  T* __restrict__ DV = static_cast<T*>(p.dv_out);
  const bool vqk = p.vec_qk, vv = p.vec_v;
  const int64_t qoff = (int64_t)hl * p.dk, voff = (int64_t)hl * p.dv;
  const WarpRange wr = warp_range(p);

  for (int64_t j = wr.first; j < wr.last; j += wr.step) {
    const int beg = __ldg(p.col_ptr + j), end = __ldg(p.col_ptr + j + 1);
    A kr[DHT], vr[DHT], gk[DHT], gv[DHT];
#pragma unroll
    for (int t = 0; t < DHT; ++t) gk[t] = gv[t] = A(0);
    if (head_ok && end > beg) {
      load_chunk<T, DHT>(K + j * p.ldq + qoff, p.dk, vqk, kr);
      load_chunk<T, DHT>(V + j * p.ldv + voff, p.dv, vv, vr);
    } else {
#pragma unroll
      for (int t = 0; t < DHT; ++t) kr[t] = vr[t] = A(0);
    }
    // two-level sum: a fresh partial per block of kSumBlock * CHUNK edges,
    // added into the total (a degree-S hub column, e.g. a global token's
    // ~5e5 in-edges, keeps ~(block + blocks) roundings instead of ~S;
    // columns shorter than one block see the same operations as one level)
    A tk[DHT], tv[DHT];
#pragma unroll
    for (int t = 0; t < DHT; ++t) tk[t] = tv[t] = A(0);
    for (int b0 = beg; b0 < end; b0 += kSumBlock * CHUNK) {
    const int b1 = min(end, b0 + kSumBlock * CHUNK);
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) gk[t] = gv[t] = A(0);
    for (int e0 = b0; e0 < b1; e0 += CHUNK) {
      const int n = min(CHUNK, b1 - e0);
      const int my_row = lane < n ? __ldg(p.csc_row + e0 + lane) : 0;
      const int my_eid = lane < n ? __ldg(p.csc_eid + e0 + lane) : 0;
      const A my_b = (bias && lane < n) ? __ldg(bias + my_eid) * A(M::kLogScale) : A(0);
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int idx = u * SLOTS + slot;
        const int i = __shfl_sync(0xffffffffu, my_row, idx & 31);
        const int e = __shfl_sync(0xffffffffu, my_eid, idx & 31);
        const A b = __shfl_sync(0xffffffffu, my_b, idx & 31);
        if (idx < n && head_ok) {
          A q[DHT], d[DHT];
          load_chunk<T, DHT>(Q + (int64_t)i * p.ldq + qoff, p.dk, vqk, q);
          load_chunk<T, DHT>(DO + (int64_t)i * p.ldv + voff, p.dv, vv, d);
          const A lse = __ldg(LSE + (int64_t)i * p.H + hl);
          const A delta = __ldg(DELTA + (int64_t)i * p.H + hl);
          const A s = score_of<A, DHT>(q, kr, scale_l, b);
          const A pr = M::ex(s - lse);
          A dw = dot_chunk<A, DHT>(d, vr);
          A pw = pr;
          if (wm) {
            const A mult = __ldg(wm + (int64_t)hl * p.E + e);
            dw = M::mul(mult, dw);
            pw = pr * mult;
          }
          const A ds = pr * (dw - delta);
#pragma unroll
          for (int t = 0; t < DHT; ++t) {
            gk[t] = M::fma(ds, q[t], gk[t]);
            gv[t] = M::fma(pw, d[t], gv[t]);
          }
        }
      }
    }
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) {
        tk[t] += gk[t];
        tv[t] += gv[t];
      }
    }
    if (two_level_sums(DHT))
#pragma unroll
      for (int t = 0; t < DHT; ++t) {
        gk[t] = tk[t];
        gv[t] = tv[t];
      }
#pragma unroll
    for (int off = LPN; off < kWarp; off <<= 1)
#pragma unroll
      for (int t = 0; t < DHT; ++t) {
        gk[t] += __shfl_xor_sync(0xffffffffu, gk[t], off);
        gv[t] += __shfl_xor_sync(0xffffffffu, gv[t], off);
      }
    if (slot == 0 && head_ok) {
      const A sc = A(p.scale);
#pragma unroll
      for (int t = 0; t < DHT; ++t) gk[t] *= sc;
      store_chunk<T, DHT>(DK + j * p.ldq + qoff, p.dk, vqk, gk);
      store_chunk<T, DHT>(DV + j * p.ldv + voff, p.dv, vv, gv);
    }
  }
}

// Finite check for K/V rows that no pattern pair references (the gathers in
// the forward kernel cover every referenced row; the reference checks all).
template <typename T>
__global__ void finite_rows_kernel(const T* __restrict__ K, const T* __restrict__ V,
                                   const int32_t* __restrict__ rows, int nrows, int64_t ldq,
                                   int64_t ldv, int64_t wq, int64_t wv, int* err) {
  int bad = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t row = rows[r];
    for (int64_t t = threadIdx.x; t < wq; t += blockDim.x) bad |= isfinite(to_acc(K[row * ldq + t])) ? 0 : 2;
    for (int64_t t = threadIdx.x; t < wv; t += blockDim.x) bad |= isfinite(to_acc(V[row * ldv + t])) ? 0 : 4;
  }
  if (bad) atomicOr(err, bad);
}

}  // namespace gte_b200

// "Wide" tile kernels: the tile schedule of attn_tile.cuh with 32-byte lane
// pieces (one 256-bit LDG per lane per gathered row) and per-row padding of
// the staged edge lists. Same math, numerics and outputs as attn_tile.cuh;
// what changes is the instruction count per (edge, head), which ncu showed
// to be the binding resource of the tile kernels (profiles/r1b: issue-active
// 60-70%, ~47 lane-instructions per edge in the forward loop):
//
//   * a lane owns 32 bytes of a row: two bf16 heads (dh = 8), one f32 head
//     (dh = 8), or half an f32 head (dh = 16). Per-edge overhead (the id and
//     bias reads, the address, the loads) is paid once per 32 bytes instead
//     of once per 16, and a gather address is one IMAD.WIDE.U32 off a
//     per-lane 64-bit base;
//   * every row's staged list is padded to a multiple of EPL with copies of
//     its first neighbour and bias -inf, so p = ex2(-inf) = 0 for a pad: no
//     per-edge bounds tests, and ids/biases come in with one LDS.128 each;
//   * dbias (summed over heads, parallel.cpp:319) is reduced across a row's
//     lanes by recursive halving: EPL edge sums leave the row's lanes in
//     log2(EPL) shuffle stages, one coalesced store per lane.
//
// Dot products keep the exact operation order of Piece<T>::dot per 16-byte
// sub-piece, summed as the xor-butterfly of attn_tile.cuh would, so scores
// are bit-identical to the hub kernels (they still serve rows and columns
// with degree > kHubDegree): degree-1 rows keep p == 1 and ds == 0 exactly.
#pragma once

#include "attn_tile.cuh"

namespace gte_b200 {

// A lane piece of NW 32-bit words (NW = 4: 16 bytes, NW = 8: 32 bytes).
template <int NW>
struct Wn {
  uint32_t w[NW];
};

template <int NW>
__device__ __forceinline__ Wn<NW> ldgp(const char* p) {
  Wn<NW> r;
  if constexpr (NW == 8) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
  } else {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = u.x, r.w[1] = u.y, r.w[2] = u.z, r.w[3] = u.w;
  }
  return r;
}

template <int NW>
__device__ __forceinline__ void stgp(char* p, const Wn<NW>& x) {
  if constexpr (NW == 8) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x.w[0]), "r"(x.w[1]),
                 "r"(x.w[2]), "r"(x.w[3]), "r"(x.w[4]), "r"(x.w[5]), "r"(x.w[6]), "r"(x.w[7])
                 : "memory");
  } else {
    *reinterpret_cast<uint4*>(p) = make_uint4(x.w[0], x.w[1], x.w[2], x.w[3]);
  }
}

template <int NW>
__device__ __forceinline__ Wn<NW> zero_wn() {
  Wn<NW> r;
#pragma unroll
  for (int t = 0; t < NW; ++t) r.w[t] = 0u;
  return r;
}

// A lane's PB-byte piece holds HPP heads (HPP >= 1), or 1/LPH of a head.
template <typename T, int PB, int HPP>
struct Wide {
  static constexpr int NW = PB / 4;                // 32-bit words per piece
  using W = Wn<NW>;
  static constexpr int NE = PB / (int)sizeof(T);   // elements per piece
  static constexpr int HE = NE / HPP;              // elements of one head in the piece
  static constexpr int HWD = NW / HPP;             // 32-bit words of one head in the piece
  static constexpr int SUB = HWD / 4;              // 16-byte sub-pieces per head chunk
  static_assert(SUB == 1 || SUB == 2, "head chunk must be 16 or 32 bytes");

  __device__ __forceinline__ static uint4 sub(const W& a, int h, int s) {
    const int b = h * HWD + s * 4;
    return make_uint4(a.w[b], a.w[b + 1], a.w[b + 2], a.w[b + 3]);
  }
  // dot of head chunk h: Piece<T>::dot per 16-byte sub-piece, then the
  // pairwise sum the xor butterfly of head_sum<2> produces
  __device__ __forceinline__ static float dot(const W& a, const W& b, int h) {
    float s = Piece<T>::dot(sub(a, h, 0), sub(b, h, 0));
    if constexpr (SUB == 2) s = s + Piece<T>::dot(sub(a, h, 1), sub(b, h, 1));
    return s;
  }
  // acc[h*HE .. (h+1)*HE) += w * x(head chunk h)
  __device__ __forceinline__ static void axpy(float w, const W& x, int h, float (&acc)[NE]) {
    constexpr int PN = Piece<T>::N;
#pragma unroll
    for (int s = 0; s < SUB; ++s) {
      float part[PN];
#pragma unroll
      for (int t = 0; t < PN; ++t) part[t] = acc[h * HE + s * PN + t];
      Piece<T>::axpy(w, sub(x, h, s), part);
#pragma unroll
      for (int t = 0; t < PN; ++t) acc[h * HE + s * PN + t] = part[t];
    }
  }
  __device__ __forceinline__ static W pack(const float (&o)[NE]) {
    constexpr int PN = Piece<T>::N;
    W r;
#pragma unroll
    for (int s = 0; s < NW / 4; ++s) {
      float part[PN];
#pragma unroll
      for (int t = 0; t < PN; ++t) part[t] = o[s * PN + t];
      const uint4 u = Piece<T>::pack(part);
      r.w[4 * s] = u.x;
      r.w[4 * s + 1] = u.y;
      r.w[4 * s + 2] = u.z;
      r.w[4 * s + 3] = u.w;
    }
    return r;
  }
  __device__ __forceinline__ static float finite_probe(const W& x, float chk) {
#pragma unroll
    for (int s = 0; s < NW / 4; ++s)
      chk = Piece<T>::finite_probe(make_uint4(x.w[4 * s], x.w[4 * s + 1], x.w[4 * s + 2], x.w[4 * s + 3]), chk);
    return chk;
  }
};

// Lane geometry of the wide kernels: LPN lanes per row, slot = row within
// the warp, piece w of the row at byte offset 32 w; the piece's first head
// hg0 (HPP heads from it when LPH == 1; head hg0 part `part` when LPH > 1).
struct WideGeom {
  int lane, slot, w, hg0, part;
  uint32_t bo;
};

template <int PB, int HPP, int LPH, int LPN>
__device__ __forceinline__ WideGeom wide_geom() {
  WideGeom g;
  g.lane = lane_id();
  g.slot = g.lane / LPN;
  g.w = g.lane % LPN;
  g.hg0 = LPH > 1 ? g.w / LPH : g.w * HPP;
  g.part = LPH > 1 ? g.w % LPH : 0;
  g.bo = (uint32_t)(g.w * PB);
  return g;
}

// Per-tile metadata of the wide kernels (padded offsets + real degrees).
struct WideMeta {
  int row[kTileRows];
  int off[kTileRows + 1];  // padded, EPL-aligned
  int gbeg[kTileRows];
  int deg[kTileRows];
  int next;
  int pad[6];  // sizeof % 16 == 0: the staged ids/biases are read as int4/float4
};
static_assert(sizeof(WideMeta) % 16 == 0, "staged arrays must be 16-byte aligned");

constexpr size_t wide_smem_bytes() { return sizeof(WideMeta) + (size_t)(kTileCap + 16) * 8 + 16; }

struct WideSmem {
  int* cols;
  float* bias;
};

__device__ __forceinline__ WideSmem wide_carve(unsigned char* raw) {
  WideSmem s;
  s.cols = reinterpret_cast<int*>(raw + sizeof(WideMeta));
  s.bias = reinterpret_cast<float*>(s.cols + kTileCap + 16);
  return s;
}

// Stage tile blockIdx.x: row ids, padded offsets, neighbour ids + biases
// (log2 units; CSC pass: second hop through csc_eid), pads (first neighbour,
// bias -inf). Ends with a barrier; returns the tile's row count.
template <int EPL>
__device__ __forceinline__ int wide_stage(WideMeta& mt, const WideSmem& s, const int32_t* __restrict__ order,
                                          const int32_t* __restrict__ tiles, const int32_t* __restrict__ ptr,
                                          const int32_t* __restrict__ idx, const int32_t* __restrict__ eid,
                                          const float* __restrict__ bias) {
  __shared__ int wsum[kTileWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int t0 = __ldg(tiles + blockIdx.x), nrows = __ldg(tiles + blockIdx.x + 1) - t0;
  int row = 0, b = 0, d = 0;
  if (t < nrows) {
    row = __ldg(order + t0 + t);
    b = __ldg(ptr + row);
    d = __ldg(ptr + row + 1) - b;
  }
  const int pd = (d + EPL - 1) / EPL * EPL;
  int x = pd;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kTileWarps ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < kTileWarps; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kTileWarps) wsum[lane] = w;
  }
  __syncthreads();
  const int excl = x - pd + (warp ? wsum[warp - 1] : 0);
  if (t < kTileRows) {
    mt.row[t] = row;
    mt.off[t] = excl;
    mt.gbeg[t] = b;
    mt.deg[t] = d;
  }
  if (t == kTileRows - 1) mt.off[kTileRows] = excl + pd;
  __syncthreads();
  for (int r = warp; r < nrows; r += kTileWarps) {
    const int o = mt.off[r], n = mt.deg[r], gb = mt.gbeg[r];
    for (int k = lane; k < n; k += 32) {
      cp_async4(s.cols + o + k, idx + gb + k);
      if (bias) cp_async4(s.bias + o + k, eid ? static_cast<const void*>(eid + gb + k) : bias + gb + k);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  constexpr float kL2e = 1.4426950408889634f;
  for (int r = warp; r < nrows; r += kTileWarps) {
    const int o = mt.off[r], n = mt.deg[r], pe = mt.off[r + 1] - o;
    for (int k = lane; k < n; k += 32) {
      float bv = 0.f;
      if (bias) bv = eid ? __ldg(bias + reinterpret_cast<const int*>(s.bias)[o + k]) : s.bias[o + k];
      s.bias[o + k] = bv * kL2e;
    }
    if (lane < pe - n) {  // pads
      s.cols[o + n + lane] = s.cols[o];
      s.bias[o + n + lane] = SoftmaxMath<float>::neg_inf();
    }
  }
  __syncthreads();
  return nrows;
}

// Own rows of a tile, one 32-byte piece per thread: finiteness (forward) or
// an L1 prefetch (backward passes).
template <int LPN, bool kProbe, typename T, int PB>
__device__ __forceinline__ void wide_own_rows(const WideMeta& mt, int nrows, const char* A, const char* B, uint32_t rb,
                                              float& chk_a, float& chk_b) {
  using WP = Wide<T, PB, 1>;
  const int total = nrows * LPN;
  for (int x = threadIdx.x; x < total; x += kTileThreads) {
    const uint32_t c = (uint32_t)(x % LPN) * (uint32_t)PB;
    const uint32_t row = (uint32_t)mt.row[x / LPN];
    if (kProbe) {
      chk_a = WP::finite_probe(ldgp<PB / 4>(A + (uint64_t)row * rb + c), chk_a);
      chk_b = WP::finite_probe(ldgp<PB / 4>(B + (uint64_t)row * rb + c), chk_b);
    } else if (c % 128u == 0) {
      prefetch_l1(A + (uint64_t)row * rb + c);
      prefetch_l1(B + (uint64_t)row * rb + c);
    }
  }
}

__device__ __forceinline__ const char* gaddr(const char* base, uint32_t j, uint32_t rb) {
  return base + (uint64_t)j * rb;  // one IMAD.WIDE.U32
}
__device__ __forceinline__ char* gaddr(char* base, uint32_t j, uint32_t rb) { return base + (uint64_t)j * rb; }

template <int EPL>
__device__ __forceinline__ void lds_ids(const WideSmem& sm, int base, uint32_t (&j)[EPL], float (&b)[EPL]) {
  if constexpr (EPL == 4) {
    const int4 c = *reinterpret_cast<const int4*>(sm.cols + base);
    const float4 f = *reinterpret_cast<const float4*>(sm.bias + base);
    j[0] = (uint32_t)c.x, j[1] = (uint32_t)c.y, j[2] = (uint32_t)c.z, j[3] = (uint32_t)c.w;
    b[0] = f.x, b[1] = f.y, b[2] = f.z, b[3] = f.w;
  } else {
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      j[u] = (uint32_t)sm.cols[base + u];
      b[u] = sm.bias[base + u];
    }
  }
}

// ---------------------------------------------------------------------------
// Forward: O, LSE (log2 units).
template <typename T, int PB, int HPP, int LPH, int LPN, int EPL, bool WM, int MINB>
__global__ void __launch_bounds__(kTileThreads, MINB) wide_fwd_kernel(SparseArgs p) {
  using WP = Wide<T, PB, HPP>;
  using W = typename WP::W;
  using M = SoftmaxMath<float>;
  constexpr int NE = WP::NE;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideMeta& mt = *reinterpret_cast<WideMeta*>(smem_raw);
  const WideSmem sm = wide_carve(smem_raw);
  const WideGeom g = wide_geom<PB, HPP, LPH, LPN>();
  const float scale_l = float(p.scale) * M::kLogScale;
  const uint32_t rb = (uint32_t)(p.ldq * sizeof(T));  // ldq == ldv on this path
  const char* Q = static_cast<const char*>(p.q) + g.bo;
  const char* K = static_cast<const char*>(p.k) + g.bo;
  const char* Vp = static_cast<const char*>(p.v) + g.bo;
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  char* O = static_cast<char*>(p.out) + g.bo;
  float* __restrict__ LSE = static_cast<float*>(p.lse);

  const int nrows = wide_stage<EPL>(mt, sm, p.order, p.tiles, p.row_ptr, p.cols, nullptr,
                                    static_cast<const float*>(p.bias));
  float chk_q = 0.f, chk_k = 0.f, chk_v = 0.f;
  wide_own_rows<LPN, true, T, PB>(mt, nrows, static_cast<const char*>(p.k), static_cast<const char*>(p.v), rb, chk_k,
                              chk_v);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int i = -1, k = 0, d = 0, dr = 0, ob = 0, gb = 0;
  W q = zero_wn<PB / 4>();
  float m[HPP], l[HPP], acc[NE];
  auto start_row = [&](int r) {
    k = 0;
#pragma unroll
    for (int h = 0; h < HPP; ++h) m[h] = M::neg_inf(), l[h] = 0.f;
#pragma unroll
    for (int t = 0; t < NE; ++t) acc[t] = 0.f;
    if (r >= 0) {
      i = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      dr = mt.deg[r];
      gb = mt.gbeg[r];
      q = ldgp<PB / 4>(gaddr(Q, (uint32_t)i, rb));
    } else {
      i = -1;
      ob = d = dr = 0;
    }
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_row(r0 < nrows ? r0 : -1);
  }

  while (__any_sync(0xffffffffu, i >= 0)) {
    {
      // idle slots (d == 0) skip the loads and compute on stale registers;
      // their results are never stored (head_sum needs the whole warp)
      uint32_t j[EPL];
      float bl[EPL];
      W kr[EPL], vr[EPL];
      if (d > 0) {
        lds_ids<EPL>(sm, ob + k, j, bl);
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          kr[u] = ldgp<PB / 4>(gaddr(K, j[u], rb));
          vr[u] = ldgp<PB / 4>(gaddr(Vp, j[u], rb));
        }
      }
#pragma unroll
      for (int h = 0; h < HPP; ++h) {
        float s[EPL];
#pragma unroll
        for (int u = 0; u < EPL; ++u) s[u] = __fmaf_rn(head_sum<LPH>(WP::dot(q, kr[u], h)), scale_l, bl[u]);
        float mx = s[0];
#pragma unroll
        for (int u = 1; u < EPL; ++u) mx = fmaxf(mx, s[u]);
        const float m_new = fmaxf(m[h], mx);  // finite: slot 0 of a step is a real edge
        const float corr = M::ex(m[h] - m_new);
        l[h] *= corr;
#pragma unroll
        for (int t = 0; t < WP::HE; ++t) acc[h * WP::HE + t] *= corr;
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          float pr = M::ex(s[u] - m_new);
          l[h] += pr;
          if (WM) {
            const int e = gb + max(min(k + u, dr - 1), 0);
            pr *= __ldg(wm + (int64_t)(g.hg0 + h) * p.E + e);
          }
          WP::axpy(pr, vr[u], h, acc);
        }
        m[h] = m_new;
      }
    }
    k += EPL;
    const bool done = i >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
        chk_q = WP::finite_probe(q, chk_q);
        float lse[HPP];
        if (d == 0) {  // empty row: zero output (attention.cpp:119-125)
          if (p.forbid_empty && g.w == 0) atomicMin(p.err + 1, i);
#pragma unroll
          for (int t = 0; t < NE; ++t) acc[t] = 0.f;
#pragma unroll
          for (int h = 0; h < HPP; ++h) lse[h] = M::neg_inf();
        } else {
#pragma unroll
          for (int h = 0; h < HPP; ++h) {
            const float inv = __frcp_rn(l[h]);  // l == 1 (degree-1 rows) stays exact
#pragma unroll
            for (int t = 0; t < WP::HE; ++t) acc[h * WP::HE + t] *= inv;
            lse[h] = m[h] + M::lg(l[h]);
          }
        }
        stgp<PB / 4>(gaddr(O, (uint32_t)i, rb), WP::pack(acc));
        if (g.part == 0) {
          float* dst = LSE + (int64_t)i * p.H + g.hg0;
          if constexpr (HPP == 2) {
            *reinterpret_cast<float2*>(dst) = make_float2(lse[0], lse[1]);
          } else {
#pragma unroll
            for (int h = 0; h < HPP; ++h) dst[h] = lse[h];
          }
        }
      }
      const int nr = rq_.refill(done, g.lane);
      if (done) start_row(nr);
    }
  }
  int bad = (isnan(chk_q) ? 1 : 0) | (isnan(chk_k) ? 2 : 0) | (isnan(chk_v) ? 4 : 0);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && g.lane == 0) atomicOr(p.err, bad);
}

// ---------------------------------------------------------------------------
// CSR pass of the backward: delta, dQ, dbias (summed over heads); writes the
// packed (lse, delta) per (row, head) for the CSC pass.
template <typename T, int PB, int HPP, int LPH, int LPN, int EPL, bool WM, int MINB>
__global__ void __launch_bounds__(kTileThreads, MINB) wide_bwd_rows_kernel(SparseArgs p) {
  using WP = Wide<T, PB, HPP>;
  using W = typename WP::W;
  using M = SoftmaxMath<float>;
  constexpr int NE = WP::NE;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideMeta& mt = *reinterpret_cast<WideMeta*>(smem_raw);
  const WideSmem sm = wide_carve(smem_raw);
  const WideGeom g = wide_geom<PB, HPP, LPH, LPN>();
  const float scale_l = float(p.scale) * M::kLogScale;
  const uint32_t rb = (uint32_t)(p.ldq * sizeof(T));
  const char* Q = static_cast<const char*>(p.q) + g.bo;
  const char* K = static_cast<const char*>(p.k) + g.bo;
  const char* Vp = static_cast<const char*>(p.v) + g.bo;
  const char* O = static_cast<const char*>(p.o) + g.bo;
  const char* DO = static_cast<const char*>(p.dout) + g.bo;
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float* __restrict__ LSE = static_cast<const float*>(p.lse);
  float2* __restrict__ LD = static_cast<float2*>(p.lsedelta);
  char* DQ = static_cast<char*>(p.dq) + g.bo;
  float* __restrict__ DB = static_cast<float*>(p.dbias);

  const int nrows = wide_stage<EPL>(mt, sm, p.order, p.tiles, p.row_ptr, p.cols, nullptr,
                                    static_cast<const float*>(p.bias));
  float dummy_a = 0.f, dummy_b = 0.f;
  wide_own_rows<LPN, false, T, PB>(mt, nrows, static_cast<const char*>(p.k), static_cast<const char*>(p.v), rb, dummy_a,
                               dummy_b);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int i = -1, k = 0, d = 0, dr = 0, ob = 0, gb = 0;
  W q = zero_wn<PB / 4>(), dd = q, oo = q;
  float lse[HPP], delta[HPP], dq[NE];
  auto start_row = [&](int r) {
    k = 0;
#pragma unroll
    for (int t = 0; t < NE; ++t) dq[t] = 0.f;
    if (r >= 0) {
      i = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      dr = mt.deg[r];
      gb = mt.gbeg[r];
      q = ldgp<PB / 4>(gaddr(Q, (uint32_t)i, rb));
      dd = ldgp<PB / 4>(gaddr(DO, (uint32_t)i, rb));
      oo = ldgp<PB / 4>(gaddr(O, (uint32_t)i, rb));
      const float* ls = LSE + (int64_t)i * p.H + g.hg0;
#pragma unroll
      for (int h = 0; h < HPP; ++h) lse[h] = __ldg(ls + h);
    } else {
      i = -1;
      ob = d = dr = 0;
    }
  };
  // delta = dO_i . O_i per head; called by the whole warp (head_sum shuffles)
  auto row_delta = [&](bool fresh) {
#pragma unroll
    for (int h = 0; h < HPP; ++h) {
      const float x = head_sum<LPH>(WP::dot(dd, oo, h));
      if (fresh) delta[h] = x;
    }
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_row(r0 < nrows ? r0 : -1);
    row_delta(true);
  }

  while (__any_sync(0xffffffffu, i >= 0)) {
    float hs[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) hs[u] = 0.f;
    {
      uint32_t j[EPL];
      float bl[EPL];
      W kr[EPL], vr[EPL];
      if (d > 0) {
        lds_ids<EPL>(sm, ob + k, j, bl);
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          kr[u] = ldgp<PB / 4>(gaddr(K, j[u], rb));
          vr[u] = ldgp<PB / 4>(gaddr(Vp, j[u], rb));
        }
      }
      // degree-1 rows: delta := dw of the edge so ds == 0 exactly here and in
      // the CSC pass (attention.cpp:265-272)
      const bool single = dr == 1;
#pragma unroll
      for (int h = 0; h < HPP; ++h) {
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const float sc = head_sum<LPH>(WP::dot(q, kr[u], h));
          float dw = head_sum<LPH>(WP::dot(dd, vr[u], h));
          const float pr = M::ex(__fmaf_rn(sc, scale_l, bl[u]) - lse[h]);
          if (WM) dw = __fmul_rn(__ldg(wm + (int64_t)(g.hg0 + h) * p.E + gb + max(min(k + u, dr - 1), 0)), dw);
          if (u == 0 && single) delta[h] = dw;
          const float ds = single ? 0.f : pr * (dw - delta[h]);
          WP::axpy(ds, kr[u], h, dq);
          hs[u] += ds;
        }
      }
    }
    if (DB) {  // dbias_e = sum over heads (parallel.cpp:319)
      if (g.part != 0) {
#pragma unroll
        for (int u = 0; u < EPL; ++u) hs[u] = 0.f;
      }
      int which;
      bool owner;
      const float tot = EdgeReduce<EPL, LPN>::run(hs, g.w, which, owner);
      if (owner && i >= 0 && k + which < dr) DB[gb + k + which] = tot;
    }
    k += EPL;
    const bool done = i >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < NE; ++t) dq[t] *= sc;
        if (d == 0) {  // empty row: the step ran on stale registers
#pragma unroll
          for (int t = 0; t < NE; ++t) dq[t] = 0.f;
        }
        stgp<PB / 4>(gaddr(DQ, (uint32_t)i, rb), WP::pack(dq));
        if (g.part == 0) {
#pragma unroll
          for (int h = 0; h < HPP; ++h) LD[(int64_t)i * p.H + g.hg0 + h] = make_float2(lse[h], delta[h]);
        }
      }
      const int nr = rq_.refill(done, g.lane);
      if (done) start_row(nr);
      row_delta(done);
    }
  }
}

// ---------------------------------------------------------------------------
// CSC pass of the backward: dK, dV per column, no atomics.
template <typename T, int PB, int HPP, int LPH, int LPN, int EPL, bool WM, int MINB>
__global__ void __launch_bounds__(kTileThreads, MINB) wide_bwd_cols_kernel(SparseArgs p) {
  using WP = Wide<T, PB, HPP>;
  using W = typename WP::W;
  using M = SoftmaxMath<float>;
  constexpr int NE = WP::NE;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WideMeta& mt = *reinterpret_cast<WideMeta*>(smem_raw);
  const WideSmem sm = wide_carve(smem_raw);
  const WideGeom g = wide_geom<PB, HPP, LPH, LPN>();
  const float scale_l = float(p.scale) * M::kLogScale;
  const uint32_t rb = (uint32_t)(p.ldq * sizeof(T));
  const char* Q = static_cast<const char*>(p.q) + g.bo;
  const char* K = static_cast<const char*>(p.k) + g.bo;
  const char* Vp = static_cast<const char*>(p.v) + g.bo;
  const char* DO = static_cast<const char*>(p.dout) + g.bo;
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float2* __restrict__ LD = static_cast<const float2*>(p.lsedelta) + g.hg0;
  char* DK = static_cast<char*>(p.dk_out) + g.bo;
  char* DV = static_cast<char*>(p.dv_out) + g.bo;
  const uint32_t ldb = (uint32_t)p.H * 8u;  // bytes per row of LD

  const int nrows = wide_stage<EPL>(mt, sm, p.order_c, p.tiles_c, p.col_ptr, p.csc_row, p.csc_eid,
                                    static_cast<const float*>(p.bias));
  float dummy_a = 0.f, dummy_b = 0.f;
  wide_own_rows<LPN, false, T, PB>(mt, nrows, static_cast<const char*>(p.q), static_cast<const char*>(p.dout), rb,
                               dummy_a, dummy_b);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int j = -1, k = 0, d = 0, dr = 0, ob = 0, gb = 0;
  W kj = zero_wn<PB / 4>(), vj = kj;
  float gk[NE], gv[NE];
  auto start_col = [&](int r) {
    k = 0;
#pragma unroll
    for (int t = 0; t < NE; ++t) gk[t] = gv[t] = 0.f;
    if (r >= 0) {
      j = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      dr = mt.deg[r];
      gb = mt.gbeg[r];
      kj = ldgp<PB / 4>(gaddr(K, (uint32_t)j, rb));
      vj = ldgp<PB / 4>(gaddr(Vp, (uint32_t)j, rb));
    } else {
      j = -1;
      ob = d = dr = 0;
    }
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_col(r0 < nrows ? r0 : -1);
  }

  while (__any_sync(0xffffffffu, j >= 0)) {
    {
      uint32_t ii[EPL];
      float bl[EPL];
      W qr[EPL], dr_[EPL];
      float2 ld[EPL][HPP];
      if (d > 0) {
        lds_ids<EPL>(sm, ob + k, ii, bl);
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
        qr[u] = ldgp<PB / 4>(gaddr(Q, ii[u], rb));
        dr_[u] = ldgp<PB / 4>(gaddr(DO, ii[u], rb));
        const float2* lp = reinterpret_cast<const float2*>(gaddr(reinterpret_cast<const char*>(LD), ii[u], ldb));
        if constexpr (HPP == 2) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(lp));
          ld[u][0] = make_float2(x.x, x.y);
          ld[u][1] = make_float2(x.z, x.w);
        } else {
#pragma unroll
          for (int h = 0; h < HPP; ++h) ld[u][h] = __ldg(lp + h);
        }
        }
      }
#pragma unroll
      for (int h = 0; h < HPP; ++h) {
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const float sc = head_sum<LPH>(WP::dot(qr[u], kj, h));
          float dw = head_sum<LPH>(WP::dot(dr_[u], vj, h));
          const float pr = M::ex(__fmaf_rn(sc, scale_l, bl[u]) - ld[u][h].x);
          float pw = pr;
          if (WM) {
            const float mult =
                __ldg(wm + (int64_t)(g.hg0 + h) * p.E + __ldg(p.csc_eid + gb + max(min(k + u, dr - 1), 0)));
            dw = __fmul_rn(mult, dw);
            pw = pr * mult;
          }
          const float ds = pr * (dw - ld[u][h].y);
          WP::axpy(ds, qr[u], h, gk);
          WP::axpy(pw, dr_[u], h, gv);
        }
      }
    }
    k += EPL;
    const bool done = j >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < NE; ++t) {
          gk[t] = d == 0 ? 0.f : gk[t] * sc;  // unreferenced column: zero (stale registers)
          gv[t] = d == 0 ? 0.f : gv[t];
        }
        stgp<PB / 4>(gaddr(DK, (uint32_t)j, rb), WP::pack(gk));
        stgp<PB / 4>(gaddr(DV, (uint32_t)j, rb), WP::pack(gv));
      }
      const int nc = rq_.refill(done, g.lane);
      if (done) start_col(nc);
    }
  }
}

}  // namespace gte_b200

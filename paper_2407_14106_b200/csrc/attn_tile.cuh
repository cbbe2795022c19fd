// "Tile" schedule for the sparse graph-attention kernels (aligned f32/bf16
// shapes; same math, numerics and outputs as attn_rowslot.cuh / attn_fast.cuh).
//
// ncu on the row-slot kernels (profiles/r1): long-scoreboard stalls ~65-70%,
// DRAM 6-14% and L2 15-29% of peak, 25-45 warp-instructions per edge. Every
// row paid a chain of dependent global round trips (row id -> row_ptr ->
// cols -> K/V), the gathers had almost no L1 reuse (rows of one cluster ran
// in input order) and the inner loop carried hub/dropout/tail handling.
//
// Execution plan (built once per pattern on the host, csrc/capi.cu
// build_exec): rows are listed in the execution order (community schedule of
// csrc/schedule.cpp, or natural), cut into tiles of <= kTileRows rows and
// <= kTileCap edges, longest rows first inside a tile; rows longer than
// kHubDegree are listed separately (hub kernels below). The CSC pass has its
// own order, tiles and hubs over columns.
//
//   stage  (all threads, once per tile): row ids and extents, a block scan of
//          the degrees, the tile's neighbour ids and biases copied to shared
//          memory with cp.async (no register cost, all in flight together),
//          biases pre-scaled to log2 units, padding slots. The tile's own K/V
//          rows (Q/dO for the CSC pass) are read once with wide loads — the
//          forward checks their finiteness there — which also pulls the
//          community's rows into L1 just before the gathers ask for them.
//   compute: SLOTS = 32/LPN rows per warp, one per slot of LPN lanes (a lane =
//          one 16-byte piece of one head), EPL edges per step, online softmax
//          per slot, no per-edge branches; a finished slot takes the next tile
//          row from a shared counter.
//
// Hub rows/columns (degree > kHubDegree, e.g. a global token attending to
// the whole sequence, proj/src/model.cpp:349-357): one CTA per hub; every
// slot of the CTA takes a strided share of the edges with its own (m, l, acc)
// (forward) or partial sums (backward), merged through shared memory.
#pragma once

#include <type_traits>

#include "attn_piece.cuh"

namespace gte_b200 {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
#ifndef GTE_TILE_ROWS
#define GTE_TILE_ROWS 128
#endif
#ifndef GTE_TILE_CAP
#define GTE_TILE_CAP 4096
#endif
constexpr int kTileRows = GTE_TILE_ROWS;  // rows (columns) per tile, <= kTileThreads
constexpr int kTileCap = GTE_TILE_CAP;    // staged edges per tile (32 KB of ids + biases at 4096)
constexpr int kTilePad = 16;      // padding slots after the staged edges (>= EPL)
constexpr int kHubDegree = 1024;  // longer rows/columns go to the hub kernels
#ifndef GTE_TILE_EPL
#define GTE_TILE_EPL 4
#endif
#ifndef GTE_TILE_MINB
#define GTE_TILE_MINB 4
#endif
#ifndef GTE_TILE_MINB_COLS
#define GTE_TILE_MINB_COLS 4
#endif
constexpr int kTileEpl = GTE_TILE_EPL;  // edges per slot per step

struct TileMeta {
  int row[kTileRows];      // row (column) id
  int off[kTileRows + 1];  // tile-local edge offsets (exclusive scan of degrees)
  int gbeg[kTileRows];     // first edge in the CSR (CSC) arrays
  int next;                // slot refill counter
  int pad[2];
};

// neighbour ids + biases (log2 units) of the staged edges; no more: the
// shared-memory carve-out comes out of the L1 that serves the K/V gathers
constexpr size_t tile_smem_bytes() { return sizeof(TileMeta) + (size_t)(kTileCap + kTilePad) * 8; }
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

struct TileSmem {
  int* cols;
  float* bias;
};

__device__ __forceinline__ TileSmem tile_carve(unsigned char* raw) {
  TileSmem s;
  s.cols = reinterpret_cast<int*>(raw + sizeof(TileMeta));
  s.bias = reinterpret_cast<float*>(s.cols + kTileCap + kTilePad);
  return s;
}

// Stage tile `blockIdx.x` of the pass. CSR pass: ptr = row_ptr, idx = cols,
// eid = null (bias indexed by edge) or the ECR remainder's original edge ids.
// CSC pass: ptr = col_ptr, idx = csc_row, eid = csc_eid. With eid the ids are
// staged in the bias slots and replaced by the biases they point at. Returns
// the tile's row count; ends with a barrier.
__device__ __forceinline__ int tile_stage(TileMeta& mt, const TileSmem& s, const int32_t* __restrict__ order,
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
  int x = d;
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
  const int excl = x - d + (warp ? wsum[warp - 1] : 0);
  if (t < kTileRows) {
    mt.row[t] = row;
    mt.off[t] = excl;
    mt.gbeg[t] = b;
  }
  if (t == kTileRows - 1) mt.off[kTileRows] = excl + d;
  __syncthreads();
  const int total = mt.off[kTileRows];  // <= kTileCap by construction (host)
  // neighbour ids (+ biases; CSC pass: edge ids into the bias slots first)
  for (int r = warp; r < nrows; r += kTileWarps) {
    const int o = mt.off[r], n = mt.off[r + 1] - o, gb = mt.gbeg[r];
    for (int k = lane; k < n; k += 32) {
      cp_async4(s.cols + o + k, idx + gb + k);
      if (bias) cp_async4(s.bias + o + k, eid ? static_cast<const void*>(eid + gb + k) : bias + gb + k);
    }
  }
  if (t < kTilePad) {  // padding: a valid row id, zero bias
    s.cols[total + t] = mt.row[0];
    s.bias[total + t] = 0.f;
  }
  cp_async_wait_all();
  __syncthreads();
  constexpr float kL2e = 1.4426950408889634f;
  if (bias) {
    if (eid) {  // second hop: bias[eid[e]], in log2 units
      const int* ids = reinterpret_cast<const int*>(s.bias);
      for (int k = t; k < total; k += kTileThreads) s.bias[k] = __ldg(bias + ids[k]) * kL2e;
    } else {
      for (int k = t; k < total; k += kTileThreads) s.bias[k] *= kL2e;
    }
  } else {
    for (int k = t; k < total; k += kTileThreads) s.bias[k] = 0.f;
  }
  __syncthreads();
  return nrows;
}

// One 16-byte piece per thread over the tile's own rows of two tensors:
// finiteness probe (forward) or an L1 prefetch (backward passes).
template <typename T, int LPN, bool kProbe>
__device__ __forceinline__ void tile_own_rows(const TileMeta& mt, int nrows, const char* A, uint32_t ra,
                                              const char* B, uint32_t rb, int row_bytes, float& chk_a,
                                              float& chk_b) {
  using P = Piece<T>;
  const int total = nrows * LPN;
#pragma unroll 4
  for (int x = threadIdx.x; x < total; x += kTileThreads) {
    const uint32_t c = (uint32_t)(x % LPN) * 16u;
    const uint32_t row = (uint32_t)mt.row[x / LPN];
    if ((int)c < row_bytes) {
      if (kProbe) {
        chk_a = P::finite_probe(ldg16(A, row * ra + c), chk_a);
        chk_b = P::finite_probe(ldg16(B, row * rb + c), chk_b);
      } else if (c % 128u == 0) {
        prefetch_l1(A + row * ra + c);
        prefetch_l1(B + row * rb + c);
      }
    }
  }
}

// Sum over the LPN lanes of a row of v[u] (u < EPL), recursive halving: after
// min(log2 EPL, log2 LPN) stages each lane holds the partial sum of one edge
// (index `which`); remaining stages are a plain butterfly. Lanes whose
// `owner` flag is set store.
template <int EPL, int LPN>
struct EdgeReduce {
  static constexpr int stages_split() {
    int s = 0, n = EPL, g = LPN;
    while (n > 1 && g > 1) { n >>= 1; g >>= 1; ++s; }
    return s;
  }
  __device__ __forceinline__ static float run(float (&v)[EPL], int w, int& which, bool& owner) {
    int n = EPL, base = 0;
    int o = LPN / 2;
#pragma unroll
    for (int st = 0; st < stages_split(); ++st) {
      const int half = n / 2;
      const bool upper = (w & o) != 0;
#pragma unroll
      for (int t = 0; t < EPL / 2; ++t) {
        if (t < half) {
          const float send = upper ? v[t] : v[t + half];
          const float keep = upper ? v[t + half] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (upper) base += half;
      n = half;
      o >>= 1;
    }
    float x = v[0];
#pragma unroll
    for (; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    which = base;
    // lanes sharing `which` after the butterfly: keep the one with low bits 0
    constexpr int kRest = LPN >> stages_split();  // lanes per edge after the split
    owner = (w & (kRest - 1)) == 0;
    return x;
  }
};

// ---------------------------------------------------------------------------
// Forward: O, LSE (log2 units).
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads, GTE_TILE_MINB) tile_fwd_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileMeta& mt = *reinterpret_cast<TileMeta*>(smem_raw);
  const TileSmem sm = tile_carve(smem_raw);
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  char* O = static_cast<char*>(p.out);
  float* __restrict__ LSE = static_cast<float*>(p.lse);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host
  constexpr bool kLaneBase = std::is_same<T, __nv_bfloat16>::value;
  const char* Kl = lane_base(K, g.bo);
  const char* Vl = lane_base(Vp, g.bo);

  const int nrows = tile_stage(mt, sm, p.order, p.tiles, p.row_ptr, p.cols, p.eid,
                               static_cast<const float*>(p.bias));
  float chk_q = 0.f, chk_k = 0.f, chk_v = 0.f;
  // own-row finiteness of K and V (attention.cpp:20-22): every non-hub row is
  // exactly one tile's own row (hub rows: hub kernel); Q is probed per row
  tile_own_rows<T, LPN, true>(mt, nrows, K, rq, Vp, rv, p.H * p.dk * (int)sizeof(T), chk_k, chk_v);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int i = -1, k = 0, d = 0, ob = 0, gb = 0, ninc = 0;
  uint4 q = make_uint4(0, 0, 0, 0);
  float m = M::neg_inf(), l = 0.f, acc[VW];
  auto start_row = [&](int r) {
    k = 0;
    m = M::neg_inf();
    l = 0.f;
    ninc = 0;
#pragma unroll
    for (int t = 0; t < VW; ++t) acc[t] = 0.f;
    if (r >= 0) {
      i = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      gb = mt.gbeg[r];
      q = ldg16(Q, (uint32_t)i * rq + g.bo);
      if (p.inc_ptr) {  // ECR tile partials of this row: the running state starts from them
        const int x0 = __ldg(p.inc_ptr + i), x1 = __ldg(p.inc_ptr + i + 1);
        ninc = x1 - x0;
        for (int x = x0; x < x1; ++x) {
          const float2 ml = __ldg(p.part_ml + (int64_t)x * p.H + g.hcl);
          const float mn = fmaxf(m, ml.x);
          const float fa = M::ex(m - mn), fb = M::ex(ml.x - mn);
          const float* pa = p.part_acc + (int64_t)x * p.part_d + g.hcl * p.dk + g.part * VW;
          l = l * fa + ml.y * fb;
#pragma unroll
          for (int t = 0; t < VW; ++t) acc[t] = acc[t] * fa + __ldg(pa + t) * fb;
          m = mn;
        }
      }
    } else {
      i = -1;
      ob = d = 0;
    }
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_row(r0 < nrows ? r0 : -1);
  }

  while (__any_sync(0xffffffffu, i >= 0)) {
    const int rem = d - k, base = ob + k;
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int jj = sm.cols[base + u];
      bl[u] = sm.bias[base + u];
      const uint32_t j = (uint32_t)jj;
      if constexpr (kLaneBase) {
        kr[u] = ldg16r(Kl, j, rq);
        vr[u] = ldg16r(Vl, j, rv);
      } else {
        kr[u] = ldg16(K, j * rq + g.bo);
        vr[u] = ldg16(Vp, j * rv + g.bo);
      }
    }
    float s[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float full = head_sum<LPH>(P::dot(q, kr[u]));
      s[u] = (u < rem) ? __fmaf_rn(full, scale_l, bl[u]) : M::neg_inf();
    }
    float mx = s[0];
#pragma unroll
    for (int u = 1; u < EPL; ++u) mx = fmaxf(mx, s[u]);
    const float m_new = fmaxf(m, mx);
    const float m_use = (m_new == M::neg_inf()) ? 0.f : m_new;
    const float corr = M::ex(m - m_use);
    l *= corr;
    scale_pairs(acc, corr);
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      float pr = M::ex(s[u] - m_use);
      l += pr;
      if (WM && u < rem) pr *= __ldg(wm + (int64_t)g.hcl * p.E + (p.eid ? __ldg(p.eid + gb + k + u) : gb + k + u));
      P::axpy_w(pr, vr[u], acc);
    }
    m = m_new;
    k += EPL;
    const bool done = i >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done) {
        if (g.head_ok) chk_q = P::finite_probe(q, chk_q);
        if (d == 0 && ninc == 0) {  // empty row: zero output (attention.cpp:119-125)
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
      const int nr = rq_.refill(done, g.lane);
      if (done) start_row(nr);
    }
  }
  int bad = (isnan(chk_q) ? 1 : 0) | (isnan(chk_k) ? 2 : 0) | (isnan(chk_v) ? 4 : 0);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && g.lane == 0) atomicOr(p.err, bad);
}

// ---------------------------------------------------------------------------
// CSR pass of the backward: delta, dQ, dbias (summed over heads). Writes the
// packed (lse, delta) pair per (row, head) for the CSC pass.
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads, GTE_TILE_MINB) tile_bwd_rows_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileMeta& mt = *reinterpret_cast<TileMeta*>(smem_raw);
  const TileSmem sm = tile_carve(smem_raw);
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const char* O = static_cast<const char*>(p.o);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float* __restrict__ LSE = static_cast<const float*>(p.lse);
  float2* __restrict__ LD = static_cast<float2*>(p.lsedelta);
  char* DQ = static_cast<char*>(p.dq);
  float* __restrict__ DB = static_cast<float*>(p.dbias);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host

  const int nrows = tile_stage(mt, sm, p.order, p.tiles, p.row_ptr, p.cols, p.eid,
                               static_cast<const float*>(p.bias));
  float dummy_a = 0.f, dummy_b = 0.f;
  tile_own_rows<T, LPN, false>(mt, nrows, K, rq, Vp, rv, p.H * p.dk * (int)sizeof(T), dummy_a, dummy_b);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int i = -1, k = 0, d = 0, ob = 0, gb = 0, ninc = 0;
  uint4 q = make_uint4(0, 0, 0, 0), dd = q, oo = q;
  float lse = 0.f, delta = 0.f, dq[VW];
  auto start_row = [&](int r) {
    k = 0;
#pragma unroll
    for (int t = 0; t < VW; ++t) dq[t] = 0.f;
    if (r >= 0) {
      i = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      gb = mt.gbeg[r];
      ninc = p.inc_ptr ? __ldg(p.inc_ptr + i + 1) - __ldg(p.inc_ptr + i) : 0;
      q = ldg16(Q, (uint32_t)i * rq + g.bo);
      dd = ldg16(DO, (uint32_t)i * rv + g.bo);
      oo = ldg16(O, (uint32_t)i * rv + g.bo);
      lse = __ldg(LSE + (int64_t)i * p.H + g.hcl);
    } else {
      i = -1;
      ob = d = 0;
    }
  };
  // delta = dO_i . O_i per head; warp-uniform call (head_sum shuffles)
  auto row_delta = [&](bool fresh) {
    const float x = head_sum<LPH>(P::dot(dd, oo));
    if (fresh) delta = x;
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_row(r0 < nrows ? r0 : -1);
    row_delta(true);
  }

  while (__any_sync(0xffffffffu, i >= 0)) {
    const int rem = d - k, base = ob + k;
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int jj = sm.cols[base + u];
      bl[u] = sm.bias[base + u];
      const uint32_t j = (uint32_t)jj;
      kr[u] = ldg16(K, j * rq + g.bo);
      vr[u] = ldg16(Vp, j * rv + g.bo);
    }
    const bool single = d == 1 && ninc == 0;
    // delta = dO_i . O_i is set at row start (row_delta); degree-1 rows take
    // the dw of their edge so ds == 0 exactly in both passes
    // (attention.cpp:265-272)
    float hs[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(q, kr[u]));
      float dw = head_sum<LPH>(P::dot(dd, vr[u]));
      const float pr = M::ex(__fmaf_rn(sc, scale_l, bl[u]) - lse);
      if (WM && u < rem) dw = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + (p.eid ? __ldg(p.eid + gb + k + u) : gb + k + u)), dw);
      if (u == 0 && single && k == 0) delta = dw;
      const float ds = (u < rem && !single) ? pr * (dw - delta) : 0.f;
      P::axpy_w(ds, kr[u], dq);
      hs[u] = (g.part == 0 && g.head_ok) ? ds : 0.f;  // one contribution per head
    }
    if (DB) {  // dbias_e = sum over heads (parallel.cpp:319)
      if constexpr (LPN >= EPL) {  // recursive halving: EPL sums leave the slot's lanes at once
        int which;
        bool owner;
        const float tot = EdgeReduce<EPL, LPN>::run(hs, g.lane % LPN, which, owner);
        if (owner && i >= 0 && which < rem) DB[p.eid ? __ldg(p.eid + gb + k + which) : gb + k + which] = tot;
      } else {
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          float hsum = hs[u];
#pragma unroll
          for (int off = 1; off < LPN; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
          if (i >= 0 && u < rem && (g.lane % LPN) == 0) DB[p.eid ? __ldg(p.eid + gb + k + u) : gb + k + u] = hsum;
        }
      }
    }
    k += EPL;
    const bool done = i >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done && g.head_ok) {
        if (ninc) {  // ECR tile dQ partials, in incidence order
          const int x0 = __ldg(p.inc_ptr + i);
          for (int x = x0; x < x0 + ninc; ++x) {
            const float* pa = p.part_acc + (int64_t)x * p.part_d + g.hcl * p.dk + g.part * VW;
#pragma unroll
            for (int t = 0; t < VW; ++t) dq[t] += __ldg(pa + t);
          }
        }
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < VW; ++t) dq[t] *= sc;
        *reinterpret_cast<uint4*>(DQ + (uint32_t)i * rq + g.bo) = P::pack(dq);
        if (g.part == 0) LD[(int64_t)i * p.H + g.hl] = make_float2(lse, delta);
      }
      const int nr = rq_.refill(done, g.lane);
      if (done) start_row(nr);
      row_delta(done);
    }
  }
}

// ---------------------------------------------------------------------------
// CSC pass of the backward: dK, dV per column, no atomics.
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads, GTE_TILE_MINB_COLS) tile_bwd_cols_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileMeta& mt = *reinterpret_cast<TileMeta*>(smem_raw);
  const TileSmem sm = tile_carve(smem_raw);
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float2* __restrict__ LD = static_cast<const float2*>(p.lsedelta);
  char* DK = static_cast<char*>(p.dk_out);
  char* DV = static_cast<char*>(p.dv_out);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host

  const int nrows = tile_stage(mt, sm, p.order_c, p.tiles_c, p.col_ptr, p.csc_row, p.csc_eid,
                               static_cast<const float*>(p.bias));
  float dummy_a = 0.f, dummy_b = 0.f;
  tile_own_rows<T, LPN, false>(mt, nrows, Q, rq, DO, rv, p.H * p.dk * (int)sizeof(T), dummy_a, dummy_b);
  if (threadIdx.x == 0) mt.next = kTileWarps * SLOTS;
  __syncthreads();

  RowQueue<SLOTS, LPN> rq_{&mt.next, nrows};
  int j = -1, k = 0, d = 0, ob = 0, gb = 0;
  uint4 kj = make_uint4(0, 0, 0, 0), vj = kj;
  float gk[VW], gv[VW];
  auto start_col = [&](int r) {
    k = 0;
#pragma unroll
    for (int t = 0; t < VW; ++t) gk[t] = gv[t] = 0.f;
    if (r >= 0) {
      j = mt.row[r];
      ob = mt.off[r];
      d = mt.off[r + 1] - ob;
      gb = mt.gbeg[r];
      kj = ldg16(K, (uint32_t)j * rq + g.bo);
      vj = ldg16(Vp, (uint32_t)j * rv + g.bo);
    } else {
      j = -1;
      ob = d = 0;
    }
  };
  {
    const int r0 = (threadIdx.x >> 5) * SLOTS + g.slot;
    start_col(r0 < nrows ? r0 : -1);
  }

  while (__any_sync(0xffffffffu, j >= 0)) {
    const int rem = d - k, base = ob + k;
    uint4 qr[EPL], dr[EPL];
    float2 ld[EPL];
    float bl[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int ii = sm.cols[base + u];
      bl[u] = sm.bias[base + u];
      const uint32_t i = (uint32_t)ii;
      qr[u] = ldg16(Q, i * rq + g.bo);
      dr[u] = ldg16(DO, i * rv + g.bo);
      ld[u] = __ldg(LD + (int64_t)i * p.H + g.hcl);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(qr[u], kj));
      float dw = head_sum<LPH>(P::dot(dr[u], vj));
      float pr = (u < rem) ? M::ex(__fmaf_rn(sc, scale_l, bl[u]) - ld[u].x) : 0.f;
      float pw = pr;
      if (WM && u < rem) {
        const float mult = __ldg(wm + (int64_t)g.hcl * p.E + __ldg(p.csc_eid + gb + k + u));
        dw = __fmul_rn(mult, dw);
        pw = pr * mult;
      }
      const float ds = pr * (dw - ld[u].y);
      P::axpy_w(ds, qr[u], gk);
      P::axpy_w(pw, dr[u], gv);
    }
    k += EPL;
    const bool done = j >= 0 && k >= d;
    if (__any_sync(0xffffffffu, done)) {
      if (done && g.head_ok) {
        if (p.cinc_ptr) {  // ECR tile dK / dV partials of this column, in incidence order
          const int x1 = __ldg(p.cinc_ptr + j + 1);
          for (int x = __ldg(p.cinc_ptr + j); x < x1; ++x) {
            const int64_t o = (int64_t)x * p.part_d + g.hcl * p.dk + g.part * VW;
#pragma unroll
            for (int t = 0; t < VW; ++t) {
              gk[t] += __ldg(p.part_dk + o + t);
              gv[t] += __ldg(p.part_dv + o + t);
            }
          }
        }
        const float sc = float(p.scale);
#pragma unroll
        for (int t = 0; t < VW; ++t) gk[t] *= sc;
        *reinterpret_cast<uint4*>(DK + (uint32_t)j * rq + g.bo) = P::pack(gk);
        *reinterpret_cast<uint4*>(DV + (uint32_t)j * rv + g.bo) = P::pack(gv);
      }
      const int nc = rq_.refill(done, g.lane);
      if (done) start_col(nc);
    }
  }
}

// ===========================================================================
// Hub kernels: one CTA per hub row (column). Slot s of the CTA takes edges
// s, s + NS, s + 2 NS, ... (NS = kTileWarps * SLOTS slots), EPL at a time.

template <int LPN>
__device__ __forceinline__ int hub_slot(const FastGeom& g) {
  return (threadIdx.x >> 5) * (kWarp / LPN) + g.slot;
}

// Forward hub: per-slot online softmax, merged over slots in shared memory.
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads) hub_fwd_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int NS = kTileWarps * SLOTS;
  __shared__ float s_m[NS][LPN], s_l[NS][LPN], s_acc[NS][LPN][VW];
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* Q = static_cast<const char*>(p.q);
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host
  const int i = __ldg(p.hubs + blockIdx.x);
  const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
  const int s0 = hub_slot<LPN>(g), w = g.lane % LPN;
  const uint4 q = ldg16(Q, (uint32_t)i * rq + g.bo);
  float m = M::neg_inf(), l = 0.f, acc[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) acc[t] = 0.f;
  // warp-uniform trip count (the slots of one warp share shuffles in the
  // head sums): the warp runs while its first slot has edges; lanes past
  // the end see only masked (ok == false) edges
  for (int w0 = beg + (int)(threadIdx.x >> 5) * SLOTS; w0 < end; w0 += NS * EPL) {
    const int e0 = w0 + g.slot;
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
    bool ok[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int e = e0 + u * NS;
      ok[u] = e < end;
      const uint32_t j = (uint32_t)__ldg(p.cols + (ok[u] ? e : beg));
      const int oe = (p.eid && ok[u]) ? __ldg(p.eid + e) : e;  // original edge id
      bl[u] = (bias && ok[u]) ? __ldg(bias + oe) * M::kLogScale : 0.f;
      kr[u] = ldg16(K, j * rq + g.bo);
      vr[u] = ldg16(Vp, j * rv + g.bo);
    }
    float s[EPL], mx = M::neg_inf();
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float full = head_sum<LPH>(P::dot(q, kr[u]));
      s[u] = ok[u] ? __fmaf_rn(full, scale_l, bl[u]) : M::neg_inf();
      mx = fmaxf(mx, s[u]);
    }
    const float m_new = fmaxf(m, mx);
    const float m_use = (m_new == M::neg_inf()) ? 0.f : m_new;
    const float corr = M::ex(m - m_use);
    l *= corr;
    scale_pairs(acc, corr);
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      float pr = M::ex(s[u] - m_use);
      l += pr;
      if (WM && ok[u]) pr *= __ldg(wm + (int64_t)g.hcl * p.E + (p.eid ? __ldg(p.eid + e0 + u * NS) : e0 + u * NS));
      P::axpy_w(pr, vr[u], acc);
    }
    m = m_new;
  }
  s_m[s0][w] = m;
  s_l[s0][w] = l;
#pragma unroll
  for (int t = 0; t < VW; ++t) s_acc[s0][w][t] = acc[t];
  __syncthreads();
  if (threadIdx.x < LPN) {  // one lane per (head, piece): merge the NS partials in slot order
    float mm = M::neg_inf();
    for (int s = 0; s < NS; ++s) mm = fmaxf(mm, s_m[s][threadIdx.x]);
    const float mu = (mm == M::neg_inf()) ? 0.f : mm;
    float ll = 0.f, aa[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) aa[t] = 0.f;
    for (int s = 0; s < NS; ++s) {
      const float f = M::ex(s_m[s][threadIdx.x] - mu);
      ll += f * s_l[s][threadIdx.x];
#pragma unroll
      for (int t = 0; t < VW; ++t) aa[t] += f * s_acc[s][threadIdx.x][t];
    }
    const FastGeom g0 = fast_geom<T, LPH, LPN>(p.H, p.dk);  // threadIdx.x < LPN: slot 0
    if (g0.head_ok) {
      const float inv = __frcp_rn(ll);
#pragma unroll
      for (int t = 0; t < VW; ++t) aa[t] *= inv;
      *reinterpret_cast<uint4*>(static_cast<char*>(p.out) + (uint32_t)i * rv + g0.bo) = P::pack(aa);
      if (g0.part == 0) static_cast<float*>(p.lse)[(int64_t)i * p.H + g0.hl] = mm + M::lg(ll);
    }
  }
  // own-row finiteness of Q, K, V of the hub row
  if (threadIdx.x < LPN && g.head_ok) {
    float c = P::finite_probe(q, 0.f), ck = P::finite_probe(ldg16(K, (uint32_t)i * rq + g.bo), 0.f),
          cv = P::finite_probe(ldg16(Vp, (uint32_t)i * rv + g.bo), 0.f);
    const int bad = (isnan(c) ? 1 : 0) | (isnan(ck) ? 2 : 0) | (isnan(cv) ? 4 : 0);
    if (bad) atomicOr(p.err, bad);
  }
}

// Backward hub, CSR side: delta, dQ (summed over slots), dbias per edge.
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads) hub_bwd_rows_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int NS = kTileWarps * SLOTS;
  __shared__ float s_acc[NS][LPN][VW];
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* K = static_cast<const char*>(p.k);
  const char* Vp = static_cast<const char*>(p.v);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  float* __restrict__ DB = static_cast<float*>(p.dbias);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host
  const int i = __ldg(p.hubs + blockIdx.x);
  const int beg = __ldg(p.row_ptr + i), end = __ldg(p.row_ptr + i + 1);
  const int s0 = hub_slot<LPN>(g), w = g.lane % LPN;
  const uint4 q = ldg16(static_cast<const char*>(p.q), (uint32_t)i * rq + g.bo);
  const uint4 dd = ldg16(static_cast<const char*>(p.dout), (uint32_t)i * rv + g.bo);
  const uint4 oo = ldg16(static_cast<const char*>(p.o), (uint32_t)i * rv + g.bo);
  const float lse = __ldg(static_cast<const float*>(p.lse) + (int64_t)i * p.H + g.hcl);
  const float delta = head_sum<LPH>(P::dot(dd, oo));  // hub rows have degree > 1
  float dq[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) dq[t] = 0.f;
  // warp-uniform trip count (the slots of one warp share shuffles in the
  // head sums): the warp runs while its first slot has edges; lanes past
  // the end see only masked (ok == false) edges
  for (int w0 = beg + (int)(threadIdx.x >> 5) * SLOTS; w0 < end; w0 += NS * EPL) {
    const int e0 = w0 + g.slot;
    uint4 kr[EPL], vr[EPL];
    float bl[EPL];
    bool ok[EPL];
    int oe[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int e = e0 + u * NS;
      ok[u] = e < end;
      const uint32_t j = (uint32_t)__ldg(p.cols + (ok[u] ? e : beg));
      oe[u] = (p.eid && ok[u]) ? __ldg(p.eid + e) : e;  // original edge id
      bl[u] = (bias && ok[u]) ? __ldg(bias + oe[u]) * M::kLogScale : 0.f;
      kr[u] = ldg16(K, j * rq + g.bo);
      vr[u] = ldg16(Vp, j * rv + g.bo);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(q, kr[u]));
      float dw = head_sum<LPH>(P::dot(dd, vr[u]));
      const float pr = M::ex(__fmaf_rn(sc, scale_l, bl[u]) - lse);
      if (WM && ok[u]) dw = __fmul_rn(__ldg(wm + (int64_t)g.hcl * p.E + oe[u]), dw);
      const float ds = ok[u] ? pr * (dw - delta) : 0.f;
      P::axpy_w(ds, kr[u], dq);
      float hsum = (g.part == 0 && g.head_ok) ? ds : 0.f;
#pragma unroll
      for (int off = LPH; off < LPN; off <<= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, off);
      if (DB && ok[u] && (g.lane % LPN) == 0) DB[oe[u]] = hsum;
    }
  }
#pragma unroll
  for (int t = 0; t < VW; ++t) s_acc[s0][w][t] = dq[t];
  __syncthreads();
  if (threadIdx.x < LPN) {
    float aa[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) aa[t] = 0.f;
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int t = 0; t < VW; ++t) aa[t] += s_acc[s][threadIdx.x][t];
    if (g.head_ok) {
      const float sc = float(p.scale);
#pragma unroll
      for (int t = 0; t < VW; ++t) aa[t] *= sc;
      *reinterpret_cast<uint4*>(static_cast<char*>(p.dq) + (uint32_t)i * rq + g.bo) = P::pack(aa);
      if (g.part == 0) static_cast<float2*>(p.lsedelta)[(int64_t)i * p.H + g.hl] = make_float2(lse, delta);
    }
  }
}

// Backward hub, CSC side: dK, dV of a hub column (summed over slots).
template <typename T, int LPH, int LPN, int EPL, bool WM>
__global__ void __launch_bounds__(kTileThreads) hub_bwd_cols_kernel(SparseArgs p) {
  using P = Piece<T>;
  using M = SoftmaxMath<float>;
  constexpr int VW = P::N;
  constexpr int SLOTS = kWarp / LPN;
  constexpr int NS = kTileWarps * SLOTS;
  __shared__ float s_k[NS][LPN][VW], s_v[NS][LPN][VW];
  const FastGeom g = fast_geom<T, LPH, LPN>(p.H, p.dk);
  const float scale_l = p.scale_l;  // float(scale) * log2(e), from the host (no per-step F2F)
  const char* Q = static_cast<const char*>(p.q);
  const char* DO = static_cast<const char*>(p.dout);
  const float* __restrict__ bias = static_cast<const float*>(p.bias);
  const float* __restrict__ wm = static_cast<const float*>(p.wmult);
  const float2* __restrict__ LD = static_cast<const float2*>(p.lsedelta);
  const uint32_t rq = p.rq_bytes, rv = p.rv_bytes;  // row strides in bytes, from the host
  const int j = __ldg(p.hubs_c + blockIdx.x);
  const int beg = __ldg(p.col_ptr + j), end = __ldg(p.col_ptr + j + 1);
  const int s0 = hub_slot<LPN>(g), w = g.lane % LPN;
  const uint4 kj = ldg16(static_cast<const char*>(p.k), (uint32_t)j * rq + g.bo);
  const uint4 vj = ldg16(static_cast<const char*>(p.v), (uint32_t)j * rv + g.bo);
  float gk[VW], gv[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) gk[t] = gv[t] = 0.f;
  // warp-uniform trip count (the slots of one warp share shuffles in the
  // head sums): the warp runs while its first slot has edges; lanes past
  // the end see only masked (ok == false) edges
  for (int w0 = beg + (int)(threadIdx.x >> 5) * SLOTS; w0 < end; w0 += NS * EPL) {
    const int e0 = w0 + g.slot;
    uint4 qr[EPL], dr[EPL];
    float2 ld[EPL];
    float bl[EPL];
    int eid[EPL];
    bool ok[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int e = e0 + u * NS;
      ok[u] = e < end;
      const int ec = ok[u] ? e : beg;
      const uint32_t i = (uint32_t)__ldg(p.csc_row + ec);
      eid[u] = __ldg(p.csc_eid + ec);
      bl[u] = (bias && ok[u]) ? __ldg(bias + eid[u]) * M::kLogScale : 0.f;
      qr[u] = ldg16(Q, i * rq + g.bo);
      dr[u] = ldg16(DO, i * rv + g.bo);
      ld[u] = __ldg(LD + (int64_t)i * p.H + g.hcl);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const float sc = head_sum<LPH>(P::dot(qr[u], kj));
      float dw = head_sum<LPH>(P::dot(dr[u], vj));
      const float pr = ok[u] ? M::ex(__fmaf_rn(sc, scale_l, bl[u]) - ld[u].x) : 0.f;
      float pw = pr;
      if (WM && ok[u]) {
        const float mult = __ldg(wm + (int64_t)g.hcl * p.E + eid[u]);
        dw = __fmul_rn(mult, dw);
        pw = pr * mult;
      }
      const float ds = pr * (dw - ld[u].y);
      P::axpy_w(ds, qr[u], gk);
      P::axpy_w(pw, dr[u], gv);
    }
  }
#pragma unroll
  for (int t = 0; t < VW; ++t) {
    s_k[s0][w][t] = gk[t];
    s_v[s0][w][t] = gv[t];
  }
  __syncthreads();
  if (threadIdx.x < LPN) {
    float ak[VW], av[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) ak[t] = av[t] = 0.f;
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        ak[t] += s_k[s][threadIdx.x][t];
        av[t] += s_v[s][threadIdx.x][t];
      }
    if (g.head_ok) {
      const float sc = float(p.scale);
#pragma unroll
      for (int t = 0; t < VW; ++t) ak[t] *= sc;
      *reinterpret_cast<uint4*>(static_cast<char*>(p.dk_out) + (uint32_t)j * rq + g.bo) = P::pack(ak);
      *reinterpret_cast<uint4*>(static_cast<char*>(p.dv_out) + (uint32_t)j * rv + g.bo) = P::pack(av);
    }
  }
}

}  // namespace gte_b200

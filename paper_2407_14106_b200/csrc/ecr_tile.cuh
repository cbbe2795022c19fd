// Elastic Computation Reformation on the tensor pipe: the dense d_b x d_b
// (= 16 x 16) sub-blocks of a cluster-sparse layout (reference
// proj/src/reformation.cpp:111-195; tile spans :176-189) run as dense tiles
// on mma.sync, while the rest of the pattern (the "remainder") stays on the
// sparse gather kernels of attn_tile.cuh. Results are merged exactly like
// one more chunk of the online softmax: per (row, head) the tile kernel
// leaves an unnormalised partial (m, l, acc) that the sparse CSR pass folds
// into its running state; the backward leaves dQ partials per row incidence
// and dK/dV partials per column incidence that the sparse CSR/CSC passes add
// in a fixed order (no atomics, deterministic).
//
// One warp owns one sub-block: its 16 Q rows, 16 K rows and 16 V rows (plus
// dO and O in the backward) are copied to shared memory with cp.async
// (16-byte chunks, XOR-swizzled so ldmatrix is conflict-free), the operand
// fragments come from ldmatrix (.trans for the value-side B operands, and
// movmatrix turns the P / dS accumulators into the transposed A operand of
// the dK / dV products). Per head h (dh = 8 or 16):
//   S  = Q_h K_h^T                  2 x m16n8k{8,16}     (16 rows x 16 cols)
//   P  = exp2(S * scale*log2e + bias*log2e - m)          online partial (fwd)
//   O  = P V_h                      dh/8 x m16n8k16
// backward:  dP = dO_h V_h^T, dS = P (dP - delta), dQ = dS K_h, dV = P^T dO_h,
// dK = dS^T Q_h, dbias_e = sum_h dS (written straight to the pair's slot).
//
// Why mma.sync and not tcgen05: a sub-block is 16 rows, and tcgen05's
// smallest M is 64; stacking four sub-blocks (different K/V columns) would
// make the products block-diagonal (>= 4x waste) and add TMEM round trips for
// a 16 x 16 x 8 product. m16n8k8 / m16n8k16 match the sub-block exactly, so
// every tensor-core product is a useful one (profiles/r2b: measured HMMA rate
// 0.46 warp-MMA/clk/SM, i.e. ~1 us for all of C3's 5453 sub-blocks).
#pragma once

#include "attn_piece.cuh"

namespace gte_b200 {

constexpr int kEcrDb = 16;       // sub-block side the kernels execute
constexpr int kEcrWarps = 4;     // sub-blocks (warps) per CTA

struct EcrArgs {
  int n_blocks = 0;
  int H = 8, dh = 8;
  int64_t E = 0;
  int64_t ldq = 0, ldv = 0;
  float scale = 1.f;                    // 1/sqrt(dh)
  const int32_t* blk = nullptr;         // [n_blocks][2] global (row0, col0)
  const int32_t* ebase = nullptr;       // [n_blocks][16] CSR index of (row0 + r, col0)
  const int32_t* inc = nullptr;         // [n_blocks][16] row incidence id of row r
  const int32_t* cinc = nullptr;        // [n_blocks][16] column incidence id of column c
  const void* q = nullptr;
  const void* k = nullptr;
  const void* v = nullptr;
  const void* o = nullptr;
  const void* dout = nullptr;
  const float* bias = nullptr;          // [E] or null
  const float* wmult = nullptr;         // [H][E] or null
  const float* lse = nullptr;           // [S][H] log2 units (backward)
  float2* part_ml = nullptr;            // fwd: [n_inc][H] (m, l)
  float* part_acc = nullptr;            // fwd: [n_inc][H*dh]; bwd: dQ partials
  float* part_dk = nullptr;             // bwd: [n_cinc][H*dh]
  float* part_dv = nullptr;             // bwd: [n_cinc][H*dh]
  float* dbias = nullptr;               // [E] or null
};

__device__ __forceinline__ void mma_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void mma_k16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ uint32_t movt16(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}

// A 16 x D bf16 tile in shared memory, 16-byte chunks XOR-swizzled by row.
template <int D>
struct SwTile {
  static constexpr int CH = D / 8;  // 16-byte chunks per row
  __device__ __forceinline__ static uint32_t off(int row, int ch) {
    return (uint32_t)(row * D * 2 + ((ch ^ (row & 7)) * 16));
  }
  // all 32 lanes: 16 rows (global row ids base + r) -> shared tile at `s`
  __device__ __forceinline__ static void load(uint32_t s, const char* g, uint32_t ld_bytes, int base, int lane) {
#pragma unroll
    for (int x = lane; x < 16 * CH; x += 32) {
      const int r = x / CH, ch = x % CH;
      cp_async16(s + off(r, ch), g + (size_t)(base + r) * ld_bytes + ch * 16);
    }
  }
};

template <int H, int DH>
struct EcrGeom {
  static constexpr int D = H * DH;
  static constexpr int KCH = DH / 8;  // 16-byte chunks per head
  static_assert(DH == 8 || DH == 16, "ECR tiles: head dim 8 or 16");
  static_assert(D % 16 == 0 && D <= 128, "ECR tiles: H * dh <= 128");
};

// ldmatrix row address of lane `lane` for the x4 load of matrices
// {m0..m3} = (row block rb_i, chunk ch_i): lane -> matrix lane/8, row lane%8.
// (selects, not an indexed array: no local memory)
template <int D>
__device__ __forceinline__ uint32_t x4_addr(uint32_t s, int lane, int rb0, int rb1, int rb2, int rb3, int ch0, int ch1,
                                            int ch2, int ch3) {
  const int m = lane >> 3;
  const int rb = m == 0 ? rb0 : m == 1 ? rb1 : m == 2 ? rb2 : rb3;
  const int ch = m == 0 ? ch0 : m == 1 ? ch1 : m == 2 ? ch2 : ch3;
  return s + SwTile<D>::off(rb * 8 + (lane & 7), ch);
}

// ---------------------------------------------------------------------------
// Forward: per sub-block and head, the partial (m, l, acc) of its 16 rows.
template <int H, int DH, bool WM>
__global__ void __launch_bounds__(kEcrWarps * 32) ecr_fwd_kernel(EcrArgs p) {
  using G = EcrGeom<H, DH>;
  constexpr int D = G::D;
  using M = SoftmaxMath<float>;
  extern __shared__ __align__(128) unsigned char ecr_smem[];
  auto smem = reinterpret_cast<unsigned char(*)[3][16 * D * 2]>(ecr_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, c = lane & 3;
  const int b = blockIdx.x * kEcrWarps + warp;
  if (b >= p.n_blocks) return;
  const int r0 = __ldg(p.blk + 2 * b), c0 = __ldg(p.blk + 2 * b + 1);
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem[warp][0]);
  const uint32_t sK = (uint32_t)__cvta_generic_to_shared(smem[warp][1]);
  const uint32_t sV = (uint32_t)__cvta_generic_to_shared(smem[warp][2]);
  const uint32_t rq = (uint32_t)(p.ldq * 2), rv = (uint32_t)(p.ldv * 2);
  SwTile<D>::load(sQ, static_cast<const char*>(p.q), rq, r0, lane);
  SwTile<D>::load(sK, static_cast<const char*>(p.k), rq, c0, lane);
  SwTile<D>::load(sV, static_cast<const char*>(p.v), rv, c0, lane);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncwarp();

  // pair slots of this lane: rows g, g+8; columns 2c, 2c+1, 8+2c, 9+2c
  const int e_lo = __ldg(p.ebase + b * 16 + g), e_hi = __ldg(p.ebase + b * 16 + g + 8);
  float bl[2][4];
  {
    const float* bs = p.bias;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const int e = hi ? e_hi : e_lo;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int col = (t >> 1) * 8 + 2 * c + (t & 1);
        bl[hi][t] = bs ? __ldg(bs + e + col) * M::kLogScale : 0.f;
      }
    }
  }
  const int i_lo = __ldg(p.inc + b * 16 + g), i_hi = __ldg(p.inc + b * 16 + g + 8);
  const float scale_l = p.scale * M::kLogScale;

#pragma unroll
  for (int h = 0; h < H; ++h) {
    // S = Q_h K_h^T, two n-tiles of 8 columns
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if constexpr (DH == 8) {
      uint32_t a[4], kb[4];
      ldsm_x4(a, x4_addr<D>(sQ, lane, 0, 1, 0, 1, h, h, h, h));
      ldsm_x4(kb, x4_addr<D>(sK, lane, 0, 1, 0, 1, h, h, h, h));
      mma_k8(s[0], a[0], a[1], kb[0]);
      mma_k8(s[1], a[0], a[1], kb[1]);
    } else {
      uint32_t a[4], kb[4];
      ldsm_x4(a, x4_addr<D>(sQ, lane, 0, 1, 0, 1, 2 * h, 2 * h, 2 * h + 1, 2 * h + 1));
      ldsm_x4(kb, x4_addr<D>(sK, lane, 0, 0, 1, 1, 2 * h, 2 * h + 1, 2 * h, 2 * h + 1));
      mma_k16(s[0], a, kb[0], kb[1]);
      mma_k16(s[1], a, kb[2], kb[3]);
    }
    // online partial per row (rows g: regs 0,1; rows g+8: regs 2,3)
    float x[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) x[nt][j] = __fmaf_rn(s[nt][j], scale_l, bl[j >> 1][nt * 2 + (j & 1)]);
    float mx[2], l[2];
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      float m = fmaxf(fmaxf(x[0][2 * hi], x[0][2 * hi + 1]), fmaxf(x[1][2 * hi], x[1][2 * hi + 1]));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      mx[hi] = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    }
    float pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) pr[nt][j] = M::ex(x[nt][j] - mx[j >> 1]);
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      float t = (pr[0][2 * hi] + pr[0][2 * hi + 1]) + (pr[1][2 * hi] + pr[1][2 * hi + 1]);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      l[hi] = t + __shfl_xor_sync(0xffffffffu, t, 2);
    }
    if (WM) {
      const float* w = p.wmult + (int64_t)h * p.E;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int j = 0; j < 4; ++j) pr[nt][j] *= __ldg(w + ((j >> 1) ? e_hi : e_lo) + nt * 8 + 2 * c + (j & 1));
    }
    const uint32_t pa[4] = {pk_bf16(pr[0][0], pr[0][1]), pk_bf16(pr[0][2], pr[0][3]), pk_bf16(pr[1][0], pr[1][1]),
                            pk_bf16(pr[1][2], pr[1][3])};
    // O_h = P V_h, dh/8 n-tiles; B from V rows by ldmatrix.trans
#pragma unroll
    for (int nc = 0; nc < G::KCH; nc += 1) {
      uint32_t vb[4];
      const int ch = h * G::KCH + nc;
      ldsm_x4_t(vb, x4_addr<D>(sV, lane, 0, 1, 0, 1, ch, ch, ch, ch));
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      mma_k16(o, pa, vb[0], vb[1]);
      const int col = h * DH + nc * 8 + 2 * c;
      *reinterpret_cast<float2*>(p.part_acc + (int64_t)i_lo * D + col) = make_float2(o[0], o[1]);
      *reinterpret_cast<float2*>(p.part_acc + (int64_t)i_hi * D + col) = make_float2(o[2], o[3]);
    }
    if (c == 0) {
      p.part_ml[(int64_t)i_lo * H + h] = make_float2(mx[0], l[0]);
      p.part_ml[(int64_t)i_hi * H + h] = make_float2(mx[1], l[1]);
    }
  }
}

// ---------------------------------------------------------------------------
// Backward: dQ partials (rows), dK / dV partials (columns), dbias of the
// sub-block's pairs (summed over heads, final).
template <int H, int DH, bool WM>
__global__ void __launch_bounds__(kEcrWarps * 32) ecr_bwd_kernel(EcrArgs p) {
  using G = EcrGeom<H, DH>;
  constexpr int D = G::D;
  using M = SoftmaxMath<float>;
  using P = Piece<__nv_bfloat16>;
  extern __shared__ __align__(128) unsigned char ecr_smem[];
  auto smem = reinterpret_cast<unsigned char(*)[5][16 * D * 2]>(ecr_smem);
  auto s_delta = reinterpret_cast<float(*)[16][H]>(ecr_smem + kEcrWarps * 5 * 16 * D * 2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, c = lane & 3;
  const int b = blockIdx.x * kEcrWarps + warp;
  if (b >= p.n_blocks) return;
  const int r0 = __ldg(p.blk + 2 * b), c0 = __ldg(p.blk + 2 * b + 1);
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem[warp][0]);
  const uint32_t sD = (uint32_t)__cvta_generic_to_shared(smem[warp][1]);
  const uint32_t sO = (uint32_t)__cvta_generic_to_shared(smem[warp][2]);
  const uint32_t sK = (uint32_t)__cvta_generic_to_shared(smem[warp][3]);
  const uint32_t sV = (uint32_t)__cvta_generic_to_shared(smem[warp][4]);
  const uint32_t rq = (uint32_t)(p.ldq * 2), rv = (uint32_t)(p.ldv * 2);
  SwTile<D>::load(sQ, static_cast<const char*>(p.q), rq, r0, lane);
  SwTile<D>::load(sD, static_cast<const char*>(p.dout), rv, r0, lane);
  SwTile<D>::load(sO, static_cast<const char*>(p.o), rv, r0, lane);
  SwTile<D>::load(sK, static_cast<const char*>(p.k), rq, c0, lane);
  SwTile<D>::load(sV, static_cast<const char*>(p.v), rv, c0, lane);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  // delta[r][h] = dO_r[h] . O_r[h], the sparse CSR pass's own formula
  // (Piece::dot over 16-byte chunks, chunk sums in lane order)
  for (int x = lane; x < 16 * H; x += 32) {
    const int r = x / H, h = x % H;
    float dsum = 0.f;
#pragma unroll
    for (int nc = 0; nc < G::KCH; ++nc) {
      const int ch = h * G::KCH + nc;
      const uint4 dd = *reinterpret_cast<const uint4*>(smem[warp][1] + SwTile<D>::off(r, ch));
      const uint4 oo = *reinterpret_cast<const uint4*>(smem[warp][2] + SwTile<D>::off(r, ch));
      dsum = nc == 0 ? P::dot(dd, oo) : dsum + P::dot(dd, oo);
    }
    s_delta[warp][r][h] = dsum;
  }
  __syncwarp();

  const int e_lo = __ldg(p.ebase + b * 16 + g), e_hi = __ldg(p.ebase + b * 16 + g + 8);
  float bl[2][4];
#pragma unroll
  for (int hi = 0; hi < 2; ++hi)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int col = (t >> 1) * 8 + 2 * c + (t & 1);
      bl[hi][t] = p.bias ? __ldg(p.bias + (hi ? e_hi : e_lo) + col) * M::kLogScale : 0.f;
    }
  const int i_lo = __ldg(p.inc + b * 16 + g), i_hi = __ldg(p.inc + b * 16 + g + 8);
  const int j_lo = __ldg(p.cinc + b * 16 + g), j_hi = __ldg(p.cinc + b * 16 + g + 8);
  const float scale_l = p.scale * M::kLogScale;
  float db[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};

#pragma unroll
  for (int h = 0; h < H; ++h) {
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    float w[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if constexpr (DH == 8) {
      uint32_t a[4], kb[4], da[4], vb[4];
      ldsm_x4(a, x4_addr<D>(sQ, lane, 0, 1, 0, 1, h, h, h, h));
      ldsm_x4(kb, x4_addr<D>(sK, lane, 0, 1, 0, 1, h, h, h, h));
      ldsm_x4(da, x4_addr<D>(sD, lane, 0, 1, 0, 1, h, h, h, h));
      ldsm_x4(vb, x4_addr<D>(sV, lane, 0, 1, 0, 1, h, h, h, h));
      mma_k8(s[0], a[0], a[1], kb[0]);
      mma_k8(s[1], a[0], a[1], kb[1]);
      mma_k8(w[0], da[0], da[1], vb[0]);
      mma_k8(w[1], da[0], da[1], vb[1]);
    } else {
      uint32_t a[4], kb[4], da[4], vb[4];
      ldsm_x4(a, x4_addr<D>(sQ, lane, 0, 1, 0, 1, 2 * h, 2 * h, 2 * h + 1, 2 * h + 1));
      ldsm_x4(kb, x4_addr<D>(sK, lane, 0, 0, 1, 1, 2 * h, 2 * h + 1, 2 * h, 2 * h + 1));
      ldsm_x4(da, x4_addr<D>(sD, lane, 0, 1, 0, 1, 2 * h, 2 * h, 2 * h + 1, 2 * h + 1));
      ldsm_x4(vb, x4_addr<D>(sV, lane, 0, 0, 1, 1, 2 * h, 2 * h + 1, 2 * h, 2 * h + 1));
      mma_k16(s[0], a, kb[0], kb[1]);
      mma_k16(s[1], a, kb[2], kb[3]);
      mma_k16(w[0], da, vb[0], vb[1]);
      mma_k16(w[1], da, vb[2], vb[3]);
    }
    const float lse_lo = __ldg(p.lse + (int64_t)(r0 + g) * H + h), lse_hi = __ldg(p.lse + (int64_t)(r0 + g + 8) * H + h);
    const float dl_lo = s_delta[warp][g][h], dl_hi = s_delta[warp][g + 8][h];
    float pw[2][4], ds[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int hi = j >> 1;
        const float pr = M::ex(__fmaf_rn(s[nt][j], scale_l, bl[hi][nt * 2 + (j & 1)]) - (hi ? lse_hi : lse_lo));
        float dw = w[nt][j], pv = pr;
        if (WM) {
          const float mult = __ldg(p.wmult + (int64_t)h * p.E + (hi ? e_hi : e_lo) + nt * 8 + 2 * c + (j & 1));
          dw = __fmul_rn(mult, dw);
          pv = pr * mult;
        }
        ds[nt][j] = pr * (dw - (hi ? dl_hi : dl_lo));
        pw[nt][j] = pv;
        db[nt][j] += ds[nt][j];
      }
    // C-layout 8x8 blocks -> A operands: dS (rows x cols) for dQ; P^T, dS^T
    // (cols x rows, movmatrix) for dV, dK
    const uint32_t sa[4] = {pk_bf16(ds[0][0], ds[0][1]), pk_bf16(ds[0][2], ds[0][3]), pk_bf16(ds[1][0], ds[1][1]),
                            pk_bf16(ds[1][2], ds[1][3])};
    const uint32_t st[4] = {movt16(sa[0]), movt16(sa[2]), movt16(sa[1]), movt16(sa[3])};
    const uint32_t pp[4] = {pk_bf16(pw[0][0], pw[0][1]), pk_bf16(pw[0][2], pw[0][3]), pk_bf16(pw[1][0], pw[1][1]),
                            pk_bf16(pw[1][2], pw[1][3])};
    const uint32_t pt[4] = {movt16(pp[0]), movt16(pp[2]), movt16(pp[1]), movt16(pp[3])};
#pragma unroll
    for (int nc = 0; nc < G::KCH; ++nc) {
      const int ch = h * G::KCH + nc;
      const int col = h * DH + nc * 8 + 2 * c;
      uint32_t kt[4], qt[4], dt[4];
      ldsm_x4_t(kt, x4_addr<D>(sK, lane, 0, 1, 0, 1, ch, ch, ch, ch));
      ldsm_x4_t(qt, x4_addr<D>(sQ, lane, 0, 1, 0, 1, ch, ch, ch, ch));
      ldsm_x4_t(dt, x4_addr<D>(sD, lane, 0, 1, 0, 1, ch, ch, ch, ch));
      float dq[4] = {0.f, 0.f, 0.f, 0.f}, dk[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
      mma_k16(dq, sa, kt[0], kt[1]);  // rows x dims, k = columns
      mma_k16(dk, st, qt[0], qt[1]);  // columns x dims, k = rows
      mma_k16(dv, pt, dt[0], dt[1]);
      *reinterpret_cast<float2*>(p.part_acc + (int64_t)i_lo * D + col) = make_float2(dq[0], dq[1]);
      *reinterpret_cast<float2*>(p.part_acc + (int64_t)i_hi * D + col) = make_float2(dq[2], dq[3]);
      *reinterpret_cast<float2*>(p.part_dk + (int64_t)j_lo * D + col) = make_float2(dk[0], dk[1]);
      *reinterpret_cast<float2*>(p.part_dk + (int64_t)j_hi * D + col) = make_float2(dk[2], dk[3]);
      *reinterpret_cast<float2*>(p.part_dv + (int64_t)j_lo * D + col) = make_float2(dv[0], dv[1]);
      *reinterpret_cast<float2*>(p.part_dv + (int64_t)j_hi * D + col) = make_float2(dv[2], dv[3]);
    }
  }
  if (p.dbias) {  // pair slots need not be 8-byte aligned: scalar stores
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) p.dbias[((j >> 1) ? e_hi : e_lo) + nt * 8 + 2 * c + (j & 1)] = db[nt][j];
  }
}

template <int H, int DH>
constexpr size_t ecr_smem_bytes(bool bwd) {
  return bwd ? (size_t)kEcrWarps * (5 * 16 * H * DH * 2 + 16 * H * 4) : (size_t)kEcrWarps * 3 * 16 * H * DH * 2;
}

}  // namespace gte_b200

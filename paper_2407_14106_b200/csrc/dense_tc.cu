// Dense attention forward on the 5th-generation tensor cores (bf16): the
// flash-style dense layer of csrc/dense.cu with both GEMMs on tcgen05.
//
// CTA = 128 query rows x one head, 4 warps; thread t owns TMEM lane / row t.
// Per block of 128 keys:
//   1. stage K [128 keys x DKP] and V^T [DVP x 128 keys] (bf16) into shared
//      memory in the canonical K-major, no-swizzle UMMA layout (8-row x
//      16-byte core matrices; LBO = 128 B between the two 8-element k halves
//      of a core-matrix pair, SBO between 8-row groups);
//   2. one elected thread issues S = Q K^T (M = 128, N = 128, K = DKP, bf16
//      -> f32 in TMEM columns [0, 128)) and commits to an mbarrier;
//   3. every thread tcgen05.ld's its row of S (4 x 32 columns), runs the
//      online-softmax update in registers (log2 domain, ex2), writes P (bf16)
//      into shared memory (A operand, K-major);
//   4. the elected thread issues O_blk = P V (M = 128, N = DVP, K = 128) into
//      TMEM columns [0, DVP) (S is already in registers) and commits;
//   5. every thread tcgen05.ld's its O_blk row: acc = acc * corr + O_blk.
// The epilogue normalises, writes O (bf16) and LSE (f32, log2 units) exactly
// like dense.cu, so the CUDA-core backward (dense.cu) consumes it unchanged.
// Pad rows (>= s_real) attend only themselves (out = m * v_r exactly).
//
// At head_dim 8 the tensor cores are far from the bound: 128 exps per row per
// key block (MUFU) dominate, 2 MMAs per block do the 4*dh flops per pair.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

namespace {

constexpr int kM = 128;  // query rows per CTA (= TMEM lanes = threads)
constexpr int kN = 128;  // keys per block

struct TcArgs {
  int64_t S, s_real;
  int H, dk, dv;
  int64_t ldq, ldv;
  const __nv_bfloat16 *q, *k, *v;
  const float* bias;   // [S*S] or null
  const float* wmult;  // [H*S*S] or null
  __nv_bfloat16* out;
  float* lse;
  float scale_l;  // log2(e) / sqrt(dk)
  int vec;        // 16-byte row chunks: dk, dv multiples of 8, 16-byte aligned rows
};

// byte offset of element (r, kk) in a canonical K-major no-swizzle tile whose
// rows hold KW bf16 elements: core matrices of 8 rows x 8 elements (128 B)
__device__ __forceinline__ uint32_t canon(int r, int kk, int KW) {
  return (uint32_t)((r >> 3) * (KW * 16) + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
  return (1u << 4)                     // D format f32
         | (1u << 7) | (1u << 10)      // A, B bf16
         | ((uint32_t)(N >> 3) << 17)  // N
         | ((uint32_t)(M >> 4) << 24); // M; A, B K-major
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(b),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// packed f32 pairs (FFMA2 / FADD2 / FMUL2 on sm_100)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&b2);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// MN-major canonical no-swizzle layout (B operand with K = keys / queries):
// element (k index kidx, n) at (n >> 3) * 2048 + (kidx >> 3) * 128 +
// (kidx & 7) * 16 + (n & 7) * 2, descriptor (LBO 128, SBO 2048); tl() below
// produces exactly these bytes.
__host__ __device__ constexpr uint32_t instr_desc_bmn(int M, int N) { return instr_desc(M, N) | (1u << 16); }

// ---- TMA-staged operand tiles ("chunk-major"): a 128-row tile of one head is
// stored as dh/8 chunks of 2 KB, chunk c = columns [8c, 8c + 8) of the 128
// rows at 16 B per row. One TMA box {8 elements, 128 rows} lands one chunk.
// The same bytes are
//   * the canonical K-major no-swizzle layout with rows as M/N and columns as
//     K: core matrix (8 rows x 16 B) strides LBO = 2048 (along K), SBO = 128
//     (along M/N) -> kdesc();
//   * the canonical MN-major layout above with rows as K and columns as N
//     -> mndesc().
// So an operand the backward needs both ways (K for S = Q K^T and dQ = dS K;
// Q and dO in the dK/dV kernel) is staged once.
__device__ __forceinline__ uint32_t tl(int r, int kk) {
  return (uint32_t)((kk >> 3) * 2048 + r * 16 + (kk & 7) * 2);
}
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr, int kc) { return smem_desc(saddr + kc * 4096, 2048, 128); }
__device__ __forceinline__ uint64_t mndesc(uint32_t saddr, int kc) { return smem_desc(saddr + kc * 256, 128, 2048); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
// box {8 columns, 128 rows} at (column x, row y) -> 2 KB of shared memory;
// rows past the map's extent (s_real) arrive as zeros
__device__ __forceinline__ void tma_chunk(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// Stage rows [r0, r0 + 128) of head h (W valid of WP columns) chunk-major:
// vec -> one elected thread issues W/8 TMA boxes on `bar` (the caller waits
// on it); otherwise every thread copies element-wise, zero-filling.
template <int WP>
__device__ __forceinline__ void stage_tl(const CUtensorMap* tm, const __nv_bfloat16* g, int64_t ld, int h, int W,
                                         int64_t r0, int n, unsigned char* dst, uint64_t* bar, int vec, int nthreads) {
  if (vec) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, (uint32_t)(W / 8) * 2048u);
      for (int c = 0; c < W / 8; ++c) tma_chunk(dst + c * 2048, tm, h * W + c * 8, (int)r0, bar);
    }
    return;
  }
  for (int x = threadIdx.x; x < 128 * WP; x += nthreads) {
    const int r = x % 128, c = x / 128;
    const __nv_bfloat16 val = (r < n && c < W) ? g[(r0 + r) * ld + (int64_t)h * W + c] : __float2bfloat16(0.f);
    *reinterpret_cast<__nv_bfloat16*>(dst + tl(r, c)) = val;
  }
}

// zero the chunks [W/8, WP/8) of a chunk-major tile (TMA never writes them)
template <int WP>
__device__ __forceinline__ void zero_pad_chunks(unsigned char* dst, int W, int nthreads) {
  const int c0 = W / 8;
  for (int x = threadIdx.x + c0 * 128; x < (WP / 8) * 128; x += nthreads)
    *reinterpret_cast<uint4*>(dst + x * 16) = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Forward K / V block [c0, c0 + n) of head h, chunk-major: K is the K-major B
// of S = Q K^T, V the MN-major B of O = P V (keys = the MMA's K). The vector
// path is one elected thread issuing TMA boxes on `bar` (in flight while the
// previous block computes); odd head widths stage element-wise, synchronously.
template <int DKP, int DVP>
__device__ __forceinline__ void fwd_stage_kv(const TcArgs& a, const CUtensorMap* tmK, const CUtensorMap* tmV, int h,
                                             int64_t c0, int n, unsigned char* Kb, unsigned char* Vb, uint64_t* bar) {
  constexpr int kT = 2 * kM;
  if (a.vec) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, (uint32_t)(a.dk / 8 + a.dv / 8) * 2048u);
      for (int c = 0; c < a.dk / 8; ++c) tma_chunk(Kb + c * 2048, tmK, h * a.dk + c * 8, (int)c0, bar);
      for (int c = 0; c < a.dv / 8; ++c) tma_chunk(Vb + c * 2048, tmV, h * a.dv + c * 8, (int)c0, bar);
    }
    return;
  }
  stage_tl<DKP>(tmK, a.k, a.ldq, h, a.dk, c0, n, Kb, bar, 0, kT);
  stage_tl<DVP>(tmV, a.v, a.ldv, h, a.dv, c0, n, Vb, bar, 0, kT);
}

// 8 warps per 128-row tile: warps w and w + 4 share TMEM lane quadrant w & 3
// (rows 32 (w & 3) ..) and split the 128 key columns in halves; row maxima
// and sums combine through shared memory; each half accumulates half of the
// output columns. Twice the warps of a 4-warp tile at the same TMEM budget
// (128 columns per CTA, 4 CTAs per SM), for latency hiding.
template <int DKP, int DVP, bool BW>  // BW: a bias or a weight_mult is present
// 3 CTAs per SM (85 registers, no spills). With the cp.async staging 4 CTAs
// at 64 registers were 3.4 % faster for dh <= 16 (r2m); since the TMA
// staging and the one-pass softmax, 3 are 0.75 % faster (profiles/r2ay)
__global__ void __launch_bounds__(2 * kM, 3)
    dense_tc_fwd_kernel(TcArgs a, const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  constexpr int kT = 2 * kM;     // threads
  constexpr int kHalfN = kN / 2; // key columns per thread
  constexpr int kHalfV = DVP / 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* Qs = smem;                       // [128 x DKP] chunk-major
  unsigned char* Ks = Qs + kM * DKP * 2;          // 2 x [128 x DKP] chunk-major, double-buffered
  unsigned char* Vm = Ks + 2 * kN * DKP * 2;      // 2 x [128 x DVP] chunk-major (= MN-major [DVP x 128])
  unsigned char* Ps = Vm + 2 * DVP * kN * 2;      // [128 x 128]
  float* red = reinterpret_cast<float*>(Ps + kM * kN * 2);  // [2][128] partial maxima / sums
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 2 * kM);  // [0] MMA commits, [1 + b] TMA of buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 3);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);  // last block whose scores outran the running max

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;
  const int rl = quad * 32 + lane;  // row within the tile (= TMEM lane)
  const int h = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kM;
  const int64_t row = r0 + rl;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(bar + b);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.vec) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
    }
    *s_flag = -1;
  }
  for (int x = tid; x < kM * DKP; x += kT) {
    const int r = x % kM, kk = x / kM;
    const int64_t gr = r0 + r;
    __nv_bfloat16 val = __float2bfloat16(0.f);
    if (gr < a.s_real && kk < a.dk) val = a.q[gr * a.ldq + (int64_t)h * a.dk + kk];
    *reinterpret_cast<__nv_bfloat16*>(Qs + tl(r, kk)) = val;
  }
  if (a.vec) {  // the pad chunks TMA never writes
    for (int b = 0; b < 2; ++b) {
      zero_pad_chunks<DKP>(Ks + b * kN * DKP * 2, a.dk, kT);
      zero_pad_chunks<DVP>(Vm + b * DVP * kN * 2, a.dv, kT);
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_row = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(Qs), sK0 = (uint32_t)__cvta_generic_to_shared(Ks);
  const uint32_t sV0 = (uint32_t)__cvta_generic_to_shared(Vm), sP = (uint32_t)__cvta_generic_to_shared(Ps);
  constexpr uint32_t kIdS = instr_desc(kM, kN), kIdO = instr_desc_bmn(kM, DVP);

  float m = -INFINITY, l = 0.f, acc[kHalfV];
#pragma unroll
  for (int t = 0; t < kHalfV; ++t) acc[t] = 0.f;
  uint32_t phase = 0;
  const bool real = row < a.s_real;
  const int cbase = half * kHalfN;

  if (a.s_real > 0) fwd_stage_kv<DKP, DVP>(a, &tmK, &tmV, h, 0, (int)(a.s_real < kN ? a.s_real : kN), Ks, Vm, bar + 1);
  int buf = 0;
  uint32_t blk = 0;
  for (int64_t c0 = 0; c0 < a.s_real; c0 += kN, buf ^= 1, ++blk) {
    const int n = (int)(a.s_real - c0 < kN ? a.s_real - c0 : kN);
    const uint32_t sK = sK0 + (uint32_t)(buf * kN * DKP * 2), sV = sV0 + (uint32_t)(buf * DVP * kN * 2);
    if (a.vec) mbar_wait(bar + 1 + buf, (blk >> 1) & 1);  // this block's K / V (issued one block ahead)
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (c0 + kN < a.s_real) {  // next block into the other buffer (its MMAs finished last block)
      const int64_t c1 = c0 + kN;
      fwd_stage_kv<DKP, DVP>(a, &tmK, &tmV, h, c1, (int)(a.s_real - c1 < kN ? a.s_real - c1 : kN),
                             Ks + (buf ^ 1) * kN * DKP * 2, Vm + (buf ^ 1) * DVP * kN * 2, bar + 1 + (buf ^ 1));
    }
    if (tid == 0) {
#pragma unroll
      for (int kc = 0; kc < DKP / 16; ++kc) mma_bf16(tmem, kdesc(sQ, kc), kdesc(sK, kc), kIdS, kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    // Full blocks without bias / weights (all but the last key block when
    // BW is off): no per-element masks, packed FFMA2 / FADD2 (the softmax
    // passes are issue-bound; the masks were ~40 % of their instructions).
    if (!BW && n == kN) {
      // After the first block: ONE pass against the running max m (FA4's
      // conditional rescale) — p = 2^(s - m) <= 2^8 unless a score outruns m
      // by more than 8 (log2 units), in which case the whole CTA redoes the
      // block below with the exact max. Saves the max pass over TMEM and its
      // row reduction through shared memory on almost every block.
      bool fast = false;
      float corr = 1.f;
      if (blk > 0) {
        const uint64_t sc2 = pk2(a.scale_l, a.scale_l), nm2 = pk2(-m, -m);
        uint64_t l2 = pk2(0.f, 0.f);
        float mx = -INFINITY;
#pragma unroll
        for (int q4 = 0; q4 < kHalfN / 16; ++q4) {
          float v16[16];
          tmem_ld16(t_row + cbase + q4 * 16, v16);
#pragma unroll
          for (int c8 = 0; c8 < 2; ++c8) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = c8 * 8 + 2 * i;
              mx = fmaxf(mx, fmaxf(v16[j], v16[j + 1]));
              float x0, x1;
              upk2(fma2(pk2(v16[j], v16[j + 1]), sc2, nm2), x0, x1);
              const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
              l2 = add2(l2, pk2(p0, p1));
              w[i] = bf16x2(p0, p1);
            }
            *reinterpret_cast<uint4*>(Ps + canon(rl, cbase + q4 * 16 + c8 * 8, kN)) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        if (mx * a.scale_l > m + 8.f) *s_flag = (int)blk;
        fence_async_smem();
        tc_before_sync();
        __syncthreads();
        tc_after_sync();
        fast = *s_flag != (int)blk;  // CTA-uniform
        if (fast) {
          float la, lb;
          upk2(l2, la, lb);
          l += la + lb;
        }
      }
      if (!fast) {
      float mx = -INFINITY;
#pragma unroll
      for (int q4 = 0; q4 < kHalfN / 16; ++q4) {
        float v16[16];
        tmem_ld16(t_row + cbase + q4 * 16, v16);
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmaxf(mx, v16[i]);
      }
      red[half * kM + rl] = mx * a.scale_l;
      __syncthreads();
      const float mn = fmaxf(m, fmaxf(red[rl], red[kM + rl]));
      corr = ex2_approx(m - mn);
      const uint64_t sc2 = pk2(a.scale_l, a.scale_l), nm2 = pk2(-mn, -mn);
      uint64_t l2 = pk2(0.f, 0.f);
#pragma unroll
      for (int q4 = 0; q4 < kHalfN / 16; ++q4) {
        float v16[16];
        tmem_ld16(t_row + cbase + q4 * 16, v16);
#pragma unroll
        for (int c8 = 0; c8 < 2; ++c8) {
          uint32_t w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = c8 * 8 + 2 * i;
            float x0, x1;
            upk2(fma2(pk2(v16[j], v16[j + 1]), sc2, nm2), x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            l2 = add2(l2, pk2(p0, p1));
            w[i] = bf16x2(p0, p1);
          }
          *reinterpret_cast<uint4*>(Ps + canon(rl, cbase + q4 * 16 + c8 * 8, kN)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      float la, lb;
      upk2(l2, la, lb);
      l = l * corr + (la + lb);
      m = mn;
      fence_async_smem();
      tc_before_sync();
      __syncthreads();
      tc_after_sync();
      }
      if (tid == 0) {
#pragma unroll
        for (int kc = 0; kc < kN / 16; ++kc)
          mma_bf16(tmem, smem_desc(sP + kc * 256, 128, kN * 16), smem_desc(sV + kc * 256, 128, 2048), kIdO, kc > 0);
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_after_sync();
#pragma unroll
      for (int c8 = 0; c8 < kHalfV / 8; ++c8) {
        float v8[8];
        tmem_ld8(t_row + half * kHalfV + c8 * 8, v8);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[c8 * 8 + i] = fmaf(acc[c8 * 8 + i], corr, v8[i]);
      }
      // no barrier here: the next block's S MMA is issued after the barrier at
      // the top of the loop, which every thread reaches only after its O_blk
      // tcgen05.ld completed
      continue;
    }
    // pass 1: this thread's half-row maximum, combined with the partner's
    float mx = -INFINITY;
#pragma unroll
    for (int q4 = 0; q4 < kHalfN / 16; ++q4) {
      float v16[16];
      tmem_ld16(t_row + cbase + q4 * 16, v16);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = cbase + q4 * 16 + i;
        float x = v16[i];
        if (BW && a.bias) {
          x *= a.scale_l;
          if (real && c < n) x = fmaf(a.bias[row * a.S + c0 + c], 1.4426950408889634f, x);
        }
        mx = fmaxf(mx, c < n ? x : -INFINITY);
      }
    }
    if (!(BW && a.bias)) mx *= a.scale_l;
    red[half * kM + rl] = mx;
    __syncthreads();
    mx = fmaxf(red[rl], red[kM + rl]);
    const float mn = fmaxf(m, mx);
    const float corr = ex2_approx(m - mn);
    l *= corr;
    // pass 2: p for this half-row -> P (bf16), partial row sum
#pragma unroll
    for (int q4 = 0; q4 < kHalfN / 16; ++q4) {
      float v32[16];
      tmem_ld16(t_row + cbase + q4 * 16, v32);
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = c8 * 8 + 2 * i, c = cbase + q4 * 16 + j;
          float x0 = fmaf(v32[j], a.scale_l, -mn), x1 = fmaf(v32[j + 1], a.scale_l, -mn);
          if (BW && a.bias && real) {
            if (c < n) x0 = fmaf(a.bias[row * a.S + c0 + c], 1.4426950408889634f, x0);
            if (c + 1 < n) x1 = fmaf(a.bias[row * a.S + c0 + c + 1], 1.4426950408889634f, x1);
          }
          float p0 = c < n ? ex2_approx(x0) : 0.f, p1 = c + 1 < n ? ex2_approx(x1) : 0.f;
          l += p0 + p1;
          if (BW && a.wmult && real) {
            const float* wr = a.wmult + ((int64_t)h * a.S + row) * a.S + c0;
            p0 = c < n ? p0 * wr[c] : 0.f;
            p1 = c + 1 < n ? p1 * wr[c + 1] : 0.f;
          }
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          w[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(Ps + canon(rl, cbase + q4 * 16 + c8 * 8, kN)) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    m = mn;
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (tid == 0) {
#pragma unroll
      for (int kc = 0; kc < kN / 16; ++kc)
        mma_bf16(tmem, smem_desc(sP + kc * 256, 128, kN * 16), smem_desc(sV + kc * 256, 128, 2048), kIdO, kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    // this half's output columns [half * DVP/2, (half + 1) * DVP/2)
#pragma unroll
    for (int c8 = 0; c8 < kHalfV / 8; ++c8) {
      float v8[8];
      tmem_ld8(t_row + half * kHalfV + c8 * 8, v8);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[c8 * 8 + i] = fmaf(acc[c8 * 8 + i], corr, v8[i]);
    }
  }
  // epilogue: row sum = both halves' partial sums
  red[half * kM + rl] = l;
  __syncthreads();
  const float lt = red[rl] + red[kM + rl];
  if (row < a.S) {
    if (real) {
      const float inv = 1.f / lt;
#pragma unroll
      for (int t = 0; t < kHalfV; ++t) {
        const int col = half * kHalfV + t;
        if (col < a.dv) a.out[row * a.ldv + (int64_t)h * a.dv + col] = __float2bfloat16(acc[t] * inv);
      }
      if (half == 0) a.lse[row * a.H + h] = m + log2f(lt);
    } else if (half == 0) {  // pad row: attends only itself (model.cpp:400-403)
      const float mult = (BW && a.wmult) ? a.wmult[((int64_t)h * a.S + row) * a.S + row] : 1.f;
      for (int t = 0; t < a.dv; ++t) {
        const float vv = __bfloat162float(a.v[row * a.ldv + (int64_t)h * a.dv + t]);
        a.out[row * a.ldv + (int64_t)h * a.dv + t] = __float2bfloat16(mult * vv);
      }
      a.lse[row * a.H + h] = 0.f;
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// Tensor map of a [rows x cols] bf16 matrix with row stride ld (elements) and
// a {8 columns, 128 rows} box; rows past `rows` read as zeros.
bool encode_rows_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t ld) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {8, 128}, estr[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DKP, int DVP>
cudaError_t launch(const TcArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)kM * DKP * 2 + 2 * (size_t)kN * DKP * 2 + 2 * (size_t)DVP * kN * 2 +
                      (size_t)kM * kN * 2 + 2 * kM * sizeof(float) + 32;
  dim3 grid((unsigned)((a.S + kM - 1) / kM), (unsigned)a.H);
  CUtensorMap tk{}, tv{};
  if (a.vec && !(encode_rows_map(&tk, a.k, (int64_t)a.H * a.dk, a.s_real, a.ldq) &&
                 encode_rows_map(&tv, a.v, (int64_t)a.H * a.dv, a.s_real, a.ldv)))
    return cudaErrorInvalidValue;
  if (a.bias || a.wmult) {
    cudaError_t e = cudaFuncSetAttribute(dense_tc_fwd_kernel<DKP, DVP, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dense_tc_fwd_kernel<DKP, DVP, true><<<grid, 2 * kM, smem, st>>>(a, tk, tv);
  } else {
    cudaError_t e = cudaFuncSetAttribute(dense_tc_fwd_kernel<DKP, DVP, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dense_tc_fwd_kernel<DKP, DVP, false><<<grid, 2 * kM, smem, st>>>(a, tk, tv);
  }
  return cudaGetLastError();
}

template <int DKP>
cudaError_t launch_dv(const TcArgs& a, cudaStream_t st) {
  const int dvp = (a.dv + 15) / 16 * 16;
  switch (dvp) {
    case 16: return launch<DKP, 16>(a, st);
    case 32: return launch<DKP, 32>(a, st);
    case 48: return launch<DKP, 48>(a, st);
    default: return launch<DKP, 64>(a, st);
  }
}


// ===========================================================================
// Backward on tcgen05 (bf16, no weight_mult, no dbias — those take the CUDA-
// core kernels of dense.cu). FA2-style, atomic-free, two kernels:
//   dq:    per 128 query rows: S = Q K^T, p = ex2(S*scale - lse); dP = dO V^T;
//          dS = p (dP - delta) -> smem (bf16); dQ += dS K (TMEM accumulator)
//   dkdv:  per 128 keys: S^T = K Q^T, p^T; dP^T = V dO^T; dV += P^T dO,
//          dK += dS^T Q (two TMEM accumulators)
// B operands that the second GEMM needs with the key / query index as K are
// staged a second time in the canonical MN-major layout (8 k-rows x 16 B of
// n per core matrix; LBO = 128 B along k, SBO = 2048 B along n).


struct TcBwdArgs {
  int64_t S, s_real;
  int H, dk, dv;
  int64_t ldq, ldv;
  const __nv_bfloat16 *q, *k, *v, *o, *dout;
  const float* bias;  // [S*S] or null (score input only)
  const float* lse;   // [S*H] log2 units (forward)
  __nv_bfloat16 *dq, *dk_out, *dv_out;
  float* delta;  // [S*H] workspace: written by the dq kernel, read by dkdv
  float scale_l, scale;
  int vec;  // 16-byte chunk staging (dk, dv multiples of 8, 16-byte aligned rows)
};

__device__ __forceinline__ __nv_bfloat16 bz() { return __float2bfloat16(0.f); }

// Both backward kernels run 8 warps per 128-row tile: warps w and w + 4 share
// TMEM lane quadrant w & 3 and split the 128 columns of S / dP (no row
// reductions are needed in the backward: lse and delta are per row / column
// inputs); the accumulators' columns are split between the two halves.
constexpr int kBT = 2 * kM;  // threads of the backward kernels

// The CTA's own 128-row tile (loaded once), chunk-major, synchronously: one
// 16-byte chunk per step on the vector path, element-wise otherwise.
template <int WP>
__device__ __forceinline__ void stage_rows_tl(const __nv_bfloat16* g, int64_t ld, int h, int W, int64_t r0, int n,
                                              unsigned char* dst, int vec) {
  if (vec) {
    for (int x = threadIdx.x; x < 128 * (WP / 8); x += kBT) {
      const int r = x % 128, c = (x / 128) * 8;
      uint4 val = make_uint4(0, 0, 0, 0);
      if (r < n && c < W) val = __ldg(reinterpret_cast<const uint4*>(g + (r0 + r) * ld + (int64_t)h * W + c));
      *reinterpret_cast<uint4*>(dst + tl(r, c)) = val;
    }
    return;
  }
  for (int x = threadIdx.x; x < 128 * WP; x += kBT) {
    const int r = x % 128, c = x / 128;
    const __nv_bfloat16 val = (r < n && c < W) ? g[(r0 + r) * ld + (int64_t)h * W + c] : bz();
    *reinterpret_cast<__nv_bfloat16*>(dst + tl(r, c)) = val;
  }
}

__device__ __forceinline__ void cp_async4z(void* smem, const void* gmem, int src_bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}

// columns [c0, c0 + NC) of this thread's TMEM lane -> v (NC multiple of 8)
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[NC]) {
#pragma unroll
  for (int c8 = 0; c8 < NC / 8; ++c8) {
    float x[8];
    tmem_ld8(taddr + c8 * 8, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[c8 * 8 + i] = x[i];
  }
}

template <int DKP, int DVP>
__global__ void __launch_bounds__(kBT, 2)
    dense_tc_dq_kernel(TcBwdArgs a, const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  constexpr int kHN = kN / 2, kHK = DKP / 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* Qs = smem;                    // [128 x DKP] chunk-major (A of S)
  unsigned char* Ds = Qs + kM * DKP * 2;       // [128 x DVP] chunk-major (A of dP)
  // key-block operands, double-buffered, chunk-major: [K | V] per buffer
  constexpr int kKB = kN * DKP * 2 + kN * DVP * 2;
  unsigned char* KB = Ds + kM * DVP * 2;       // 2 x {K [128 keys x DKP] (K-major B of S, MN-major B of dQ),
                                               //      V [128 keys x DVP] (K-major B of dP)}
  unsigned char* dS = KB + 2 * kKB;            // [128 x 128] K-major (A of dQ)
  uint64_t* bar = reinterpret_cast<uint64_t*>(dS + kM * kN * 2);  // [0] MMA, [1 + b] TMA of buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp & 3, half = warp >> 2;
  const int rl = quad * 32 + lane, cb = half * kHN, h = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kM, row = r0 + rl;
  const bool real = row < a.s_real;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(bar + b);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.vec) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
    }
  }
  const int nq = (int)(a.s_real - r0 < kM ? (a.s_real - r0 > 0 ? a.s_real - r0 : 0) : kM);
  stage_rows_tl<DKP>(a.q, a.ldq, h, a.dk, r0, nq, Qs, a.vec);
  stage_rows_tl<DVP>(a.dout, a.ldv, h, a.dv, r0, nq, Ds, a.vec);
  if (a.vec) {
    for (int b = 0; b < 2; ++b) {
      zero_pad_chunks<DKP>(KB + b * kKB, a.dk, kBT);
      zero_pad_chunks<DVP>(KB + b * kKB + kN * DKP * 2, a.dv, kBT);
    }
  }
  float lse = 0.f, delta = 0.f;
  if (real) {
    lse = a.lse[row * a.H + h];
    for (int t = 0; t < a.dv; ++t)
      delta += __bfloat162float(a.dout[row * a.ldv + (int64_t)h * a.dv + t]) *
               __bfloat162float(a.o[row * a.ldv + (int64_t)h * a.dv + t]);
    if (half == 0) a.delta[row * a.H + h] = delta;  // for the dkdv kernel
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot, t_row = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(Qs), sD = (uint32_t)__cvta_generic_to_shared(Ds);
  const uint32_t sKB = (uint32_t)__cvta_generic_to_shared(KB), sS = (uint32_t)__cvta_generic_to_shared(dS);
  auto stage_keys = [&](int64_t c, int b) {  // one TMA barrier per buffer: K and V chunks
    const int nn = (int)(a.s_real - c < kN ? a.s_real - c : kN);
    unsigned char* base = KB + b * kKB;
    if (a.vec) {
      if (tid == 0) {
        mbar_expect_tx(bar + 1 + b, (uint32_t)(a.dk / 8 + a.dv / 8) * 2048u);
        for (int x = 0; x < a.dk / 8; ++x) tma_chunk(base + x * 2048, &tmK, h * a.dk + x * 8, (int)c, bar + 1 + b);
        for (int x = 0; x < a.dv / 8; ++x)
          tma_chunk(base + kN * DKP * 2 + x * 2048, &tmV, h * a.dv + x * 8, (int)c, bar + 1 + b);
      }
      return;
    }
    stage_tl<DKP>(&tmK, a.k, a.ldq, h, a.dk, c, nn, base, nullptr, 0, kBT);
    stage_tl<DVP>(&tmV, a.v, a.ldv, h, a.dv, c, nn, base + kN * DKP * 2, nullptr, 0, kBT);
  };
  uint32_t phase = 0;
  float g[kHK];  // this thread's half of its dQ row, summed over key blocks in registers
#pragma unroll
  for (int t = 0; t < kHK; ++t) g[t] = 0.f;
  const bool rows_full = r0 + kM <= a.s_real;  // CTA-uniform
  const uint64_t sc2 = pk2(a.scale_l, a.scale_l), nl2 = pk2(-lse, -lse), nd2 = pk2(-delta, -delta);
  if (a.s_real > 0) stage_keys(0, 0);
  int buf = 0;
  uint32_t blk = 0;
  for (int64_t c0 = 0; c0 < a.s_real; c0 += kN, buf ^= 1, ++blk) {
    const int n = (int)(a.s_real - c0 < kN ? a.s_real - c0 : kN);
    const uint32_t sK = sKB + (uint32_t)(buf * kKB), sV = sK + kN * DKP * 2;
    if (a.vec) mbar_wait(bar + 1 + buf, (blk >> 1) & 1);  // this block's keys (issued one block ahead)
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (c0 + kN < a.s_real) stage_keys(c0 + kN, buf ^ 1);  // the other buffer's MMAs completed last block
    if (tid == 0) {  // S = Q K^T -> columns [0, 128), dP = dO V^T -> [128, 256): independent, one commit
#pragma unroll
      for (int kc = 0; kc < DKP / 16; ++kc) mma_bf16(tmem, kdesc(sQ, kc), kdesc(sK, kc), instr_desc(kM, kN), kc > 0);
#pragma unroll
      for (int kc = 0; kc < DVP / 16; ++kc)
        mma_bf16(tmem + 128, kdesc(sD, kc), kdesc(sV, kc), instr_desc(kM, kN), kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    float p[kHN];
    const bool fast = !a.bias && n == kN && rows_full;
#pragma unroll
    for (int q4 = 0; q4 < kHN / 16; ++q4) {
      float v16[16];
      tmem_ld16(t_row + cb + q4 * 16, v16);
      if (fast) {  // full block, every row real, no bias: no masks, packed scale-shift
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          float x0, x1;
          upk2(fma2(pk2(v16[i], v16[i + 1]), sc2, nl2), x0, x1);
          p[q4 * 16 + i] = ex2_approx(x0);
          p[q4 * 16 + i + 1] = ex2_approx(x1);
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = cb + q4 * 16 + i;
        float x = fmaf(v16[i], a.scale_l, -lse);
        if (a.bias && real && c < n) x = fmaf(a.bias[row * a.S + c0 + c], 1.4426950408889634f, x);
        p[q4 * 16 + i] = (real && c < n) ? ex2_approx(x) : 0.f;
      }
    }
#pragma unroll
    for (int q4 = 0; q4 < kHN / 16; ++q4) {
      float v16[16];
      tmem_ld16(t_row + 128 + cb + q4 * 16, v16);
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = c8 * 8 + 2 * i, pc = q4 * 16 + j;
          float d0, d1;  // p (dP - delta), packed
          upk2(mul2(pk2(p[pc], p[pc + 1]), add2(pk2(v16[j], v16[j + 1]), nd2)), d0, d1);
          w[i] = bf16x2(d0, d1);
        }
        *reinterpret_cast<uint4*>(dS + canon(rl, cb + q4 * 16 + c8 * 8, kN)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (tid == 0) {  // dQ_blk = dS K into the consumed S columns (A = dS K-major, B = K MN-major, N = DKP)
#pragma unroll
      for (int kc = 0; kc < kN / 16; ++kc)
        mma_bf16(tmem, smem_desc(sS + kc * 256, 128, kN * 16), mndesc(sK, kc), instr_desc_bmn(kM, DKP), kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    {
      float gb[kHK];
      tmem_ld_cols<kHK>(t_row + half * kHK, gb);
#pragma unroll
      for (int t = 0; t < kHK; ++t) g[t] += gb[t];
    }
  }
  // tcgen05.ld is warp-collective: every thread loaded, only valid rows store
  if (row < a.S) {
#pragma unroll
    for (int t = 0; t < kHK; ++t) {
      const int col = half * kHK + t;
      if (col < a.dk) a.dq[row * a.ldq + (int64_t)h * a.dk + col] = __float2bfloat16(real ? g[t] * a.scale : 0.f);
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int DKP, int DVP>
__global__ void __launch_bounds__(kBT, 2)
    dense_tc_dkdv_kernel(TcBwdArgs a, const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmD) {
  constexpr int kHN = kN / 2, kHK = DKP / 2, kHV = DVP / 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* Ks = smem;                    // [128 keys x DKP] chunk-major (A of S^T)
  unsigned char* Vs = Ks + kM * DKP * 2;       // [128 keys x DVP] chunk-major (A of dP^T)
  // query-block operands, double-buffered: [Q | dO | lse | delta] per buffer
  constexpr int kQB = (kN * DKP + kN * DVP) * 2 + 2 * kN * 4;
  unsigned char* QB = Vs + kM * DVP * 2;       // 2 x {Q [128 q x DKP] chunk-major (K-major B of S^T, MN-major B of dK),
                                               //      dO [128 q x DVP] chunk-major (K-major B of dP^T, MN-major B of dV),
                                               //      lse [128], delta [128] of the query block}
  unsigned char* Pt = QB + 2 * kQB;            // [128 keys x 128 q] K-major (A of dV)
  unsigned char* St = Pt + kM * kN * 2;        // [128 keys x 128 q] K-major (A of dK)
  uint64_t* bar = reinterpret_cast<uint64_t*>(St + kM * kN * 2);  // [0] MMA, [1 + b] TMA of buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp & 3, half = warp >> 2;
  const int rl = quad * 32 + lane, cb = half * kHN, h = blockIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * kM, key = k0 + rl;
  const bool real = key < a.s_real;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(bar + b);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.vec) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmD);
    }
  }
  const int nk = (int)(a.s_real - k0 < kM ? (a.s_real - k0 > 0 ? a.s_real - k0 : 0) : kM);
  stage_rows_tl<DKP>(a.k, a.ldq, h, a.dk, k0, nk, Ks, a.vec);
  stage_rows_tl<DVP>(a.v, a.ldv, h, a.dv, k0, nk, Vs, a.vec);
  if (a.vec) {
    for (int b = 0; b < 2; ++b) {
      zero_pad_chunks<DKP>(QB + b * kQB, a.dk, kBT);
      zero_pad_chunks<DVP>(QB + b * kQB + kN * DKP * 2, a.dv, kBT);
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot, t_row = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t sK = (uint32_t)__cvta_generic_to_shared(Ks), sV = (uint32_t)__cvta_generic_to_shared(Vs);
  const uint32_t sQB = (uint32_t)__cvta_generic_to_shared(QB);
  const uint32_t sPt = (uint32_t)__cvta_generic_to_shared(Pt), sSt = (uint32_t)__cvta_generic_to_shared(St);
  constexpr uint32_t kColV = 0, kColK = DVP;  // dV_blk, dK_blk (registers accumulate them)
  constexpr int oDk = kN * DKP * 2, oLs = oDk + kN * DVP * 2;
  auto stage_queries = [&](int64_t q, int b) {
    const int nn = (int)(a.s_real - q < kN ? a.s_real - q : kN);
    unsigned char* base = QB + b * kQB;
    if (a.vec) {
      if (tid == 0) {
        mbar_expect_tx(bar + 1 + b, (uint32_t)(a.dk / 8 + a.dv / 8) * 2048u);
        for (int x = 0; x < a.dk / 8; ++x) tma_chunk(base + x * 2048, &tmQ, h * a.dk + x * 8, (int)q, bar + 1 + b);
        for (int x = 0; x < a.dv / 8; ++x)
          tma_chunk(base + oDk + x * 2048, &tmD, h * a.dv + x * 8, (int)q, bar + 1 + b);
      }
    } else {
      stage_tl<DKP>(&tmQ, a.q, a.ldq, h, a.dk, q, nn, base, nullptr, 0, kBT);
      stage_tl<DVP>(&tmD, a.dout, a.ldv, h, a.dv, q, nn, base + oDk, nullptr, 0, kBT);
    }
    if (tid < kN) {  // lse, delta (the dq kernel's dO . O) of the block's queries; zeros past the end
      const bool ok = tid < nn;
      const int64_t qr = ok ? q + tid : 0;
      float* lsb = reinterpret_cast<float*>(base + oLs);
      cp_async4z(lsb + tid, a.lse + qr * a.H + h, ok ? 4 : 0);
      cp_async4z(lsb + kN + tid, a.delta + qr * a.H + h, ok ? 4 : 0);
    }
    cp_async_commit();
  };
  uint32_t phase = 0;
  float gv[kHV], gk[kHK];  // this thread's halves of its dV / dK rows, summed over query blocks in registers
#pragma unroll
  for (int t = 0; t < kHV; ++t) gv[t] = 0.f;
#pragma unroll
  for (int t = 0; t < kHK; ++t) gk[t] = 0.f;
  const bool keys_full = k0 + kM <= a.s_real;  // CTA-uniform
  if (a.s_real > 0) stage_queries(0, 0);
  int buf = 0;
  uint32_t blk = 0;
  for (int64_t q0 = 0; q0 < a.s_real; q0 += kN, buf ^= 1, ++blk) {
    const int n = (int)(a.s_real - q0 < kN ? a.s_real - q0 : kN);
    const uint32_t sQk = sQB + (uint32_t)(buf * kQB), sDk = sQk + oDk;
    const float* ls = reinterpret_cast<const float*>(QB + buf * kQB + oLs);
    const float* dl = ls + kN;
    cp_async_wait0();                                     // this block's lse / delta
    if (a.vec) mbar_wait(bar + 1 + buf, (blk >> 1) & 1);  // and its Q / dO tiles (issued one block ahead)
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (q0 + kN < a.s_real) stage_queries(q0 + kN, buf ^ 1);  // the other buffer's MMAs completed last block
    if (tid == 0) {  // S^T = K Q^T -> columns [0, 128), dP^T = V dO^T -> [128, 256): one commit
#pragma unroll
      for (int kc = 0; kc < DKP / 16; ++kc)
        mma_bf16(tmem, kdesc(sK, kc), kdesc(sQk, kc), instr_desc(kM, kN), kc > 0);
#pragma unroll
      for (int kc = 0; kc < DVP / 16; ++kc)
        mma_bf16(tmem + 128, kdesc(sV, kc), kdesc(sDk, kc), instr_desc(kM, kN), kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    float p[kHN];
    const bool fast = !a.bias && n == kN && keys_full;
#pragma unroll
    for (int q4 = 0; q4 < kHN / 16; ++q4) {
      float v16[16];
      tmem_ld16(t_row + cb + q4 * 16, v16);
      if (fast) {  // full block, every key real, no bias: no masks
        const float4* l4 = reinterpret_cast<const float4*>(ls + cb + q4 * 16);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 lv = l4[i4];
          const int i = 4 * i4;
          p[q4 * 16 + i] = ex2_approx(fmaf(v16[i], a.scale_l, -lv.x));
          p[q4 * 16 + i + 1] = ex2_approx(fmaf(v16[i + 1], a.scale_l, -lv.y));
          p[q4 * 16 + i + 2] = ex2_approx(fmaf(v16[i + 2], a.scale_l, -lv.z));
          p[q4 * 16 + i + 3] = ex2_approx(fmaf(v16[i + 3], a.scale_l, -lv.w));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = cb + q4 * 16 + i;
          float x = fmaf(v16[i], a.scale_l, -ls[c]);
          if (a.bias && real && c < n) x = fmaf(a.bias[(q0 + c) * a.S + key], 1.4426950408889634f, x);
          p[q4 * 16 + i] = (real && c < n) ? ex2_approx(x) : 0.f;
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pc = q4 * 16 + c8 * 8 + 2 * i;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p[pc], p[pc + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(Pt + canon(rl, cb + q4 * 16 + c8 * 8, kN)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
#pragma unroll
    for (int q4 = 0; q4 < kHN / 16; ++q4) {
      float v16[16];
      tmem_ld16(t_row + 128 + cb + q4 * 16, v16);
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = c8 * 8 + 2 * i, pc = q4 * 16 + j, c = cb + pc;
          const float2 dd = *reinterpret_cast<const float2*>(dl + c);
          float d0, d1;  // p (dP - delta), packed
          upk2(mul2(pk2(p[pc], p[pc + 1]), add2(pk2(v16[j], v16[j + 1]), pk2(-dd.x, -dd.y))), d0, d1);
          w[i] = bf16x2(d0, d1);
        }
        *reinterpret_cast<uint4*>(St + canon(rl, cb + q4 * 16 + c8 * 8, kN)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (tid == 0) {  // dV_blk = P^T dO, dK_blk = dS^T Q into the consumed S^T columns
#pragma unroll
      for (int kc = 0; kc < kN / 16; ++kc)
        mma_bf16(tmem + kColV, smem_desc(sPt + kc * 256, 128, kN * 16), mndesc(sDk, kc),
                 instr_desc_bmn(kM, DVP), kc > 0);
#pragma unroll
      for (int kc = 0; kc < kN / 16; ++kc)
        mma_bf16(tmem + kColK, smem_desc(sSt + kc * 256, 128, kN * 16), mndesc(sQk, kc),
                 instr_desc_bmn(kM, DKP), kc > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_after_sync();
    {
      float bv[kHV], bk[kHK];
      tmem_ld_cols<kHV>(t_row + kColV + half * kHV, bv);
      tmem_ld_cols<kHK>(t_row + kColK + half * kHK, bk);
#pragma unroll
      for (int t = 0; t < kHV; ++t) gv[t] += bv[t];
#pragma unroll
      for (int t = 0; t < kHK; ++t) gk[t] += bk[t];
    }
  }
  // tcgen05.ld is warp-collective: every thread loaded, only valid keys store
  if (real) {
#pragma unroll
    for (int t = 0; t < kHV; ++t) {
      const int col = half * kHV + t;
      if (col < a.dv) a.dv_out[key * a.ldv + (int64_t)h * a.dv + col] = __float2bfloat16(gv[t]);
    }
#pragma unroll
    for (int t = 0; t < kHK; ++t) {
      const int col = half * kHK + t;
      if (col < a.dk) a.dk_out[key * a.ldq + (int64_t)h * a.dk + col] = __float2bfloat16(gk[t] * a.scale);
    }
  } else if (key < a.S && half == 0) {  // pad column: only its own pad row attends, p = 1: dV = dO, dK = 0
    for (int t = 0; t < a.dk; ++t) a.dk_out[key * a.ldq + (int64_t)h * a.dk + t] = bz();
    for (int t = 0; t < a.dv; ++t)
      a.dv_out[key * a.ldv + (int64_t)h * a.dv + t] = a.dout[key * a.ldv + (int64_t)h * a.dv + t];
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int DKP, int DVP>
cudaError_t launch_bwd(const TcBwdArgs& a, cudaStream_t st) {
  const size_t s1 = (size_t)kM * (DKP + DVP) * 2 + 2 * (size_t)kN * (DKP + DVP) * 2 + (size_t)kM * kN * 2 + 32;
  const size_t s2 = (size_t)kM * (DKP + DVP) * 2 + 2 * ((size_t)kN * (DKP + DVP) * 2 + 2 * kN * 4) +
                    2 * (size_t)kM * kN * 2 + 32;
  CUtensorMap tq{}, tk{}, tv{}, td{};
  if (a.vec && !(encode_rows_map(&tq, a.q, (int64_t)a.H * a.dk, a.s_real, a.ldq) &&
                 encode_rows_map(&tk, a.k, (int64_t)a.H * a.dk, a.s_real, a.ldq) &&
                 encode_rows_map(&tv, a.v, (int64_t)a.H * a.dv, a.s_real, a.ldv) &&
                 encode_rows_map(&td, a.dout, (int64_t)a.H * a.dv, a.s_real, a.ldv)))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dense_tc_dq_kernel<DKP, DVP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)s1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(dense_tc_dkdv_kernel<DKP, DVP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.S + kM - 1) / kM), (unsigned)a.H);
  dense_tc_dq_kernel<DKP, DVP><<<grid, kBT, s1, st>>>(a, tk, tv);
  dense_tc_dkdv_kernel<DKP, DVP><<<grid, kBT, s2, st>>>(a, tq, td);
  return cudaGetLastError();
}

template <int DKP>
cudaError_t launch_bwd_dv(const TcBwdArgs& a, cudaStream_t st) {
  switch ((a.dv + 15) / 16 * 16) {
    case 16: return launch_bwd<DKP, 16>(a, st);
    case 32: return launch_bwd<DKP, 32>(a, st);
    case 48: return launch_bwd<DKP, 48>(a, st);
    default: return launch_bwd<DKP, 64>(a, st);
  }
}
}  // namespace

namespace gte_b200 {

// bf16 dense forward on tcgen05 (dk, dv <= 64); the caller validated the args
cudaError_t launch_dense_tc_fwd(int64_t S, int64_t s_real, int H, int dk, int dv, const void* q, const void* k,
                                int64_t ldq, const void* v, int64_t ldv, const void* bias, const void* wmult,
                                void* out, void* lse, cudaStream_t st) {
  TcArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.bias = static_cast<const float*>(bias);
  a.wmult = static_cast<const float*>(wmult);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.lse = static_cast<float*>(lse);
  a.scale_l = (float)(1.4426950408889634 / std::sqrt((double)dk));
  a.vec = dk % 8 == 0 && dv % 8 == 0 && (ldq * 2) % 16 == 0 && (ldv * 2) % 16 == 0 &&
          (reinterpret_cast<uintptr_t>(k) % 16) == 0 && (reinterpret_cast<uintptr_t>(v) % 16) == 0;
  const int dkp = (dk + 15) / 16 * 16;
  switch (dkp) {
    case 16: return launch_dv<16>(a, st);
    case 32: return launch_dv<32>(a, st);
    case 48: return launch_dv<48>(a, st);
    default: return launch_dv<64>(a, st);
  }
}

// bf16 dense backward on tcgen05 (no weight_mult / dbias; dk, dv <= 64)
cudaError_t launch_dense_tc_bwd(int64_t S, int64_t s_real, int H, int dk, int dv, const void* q, const void* k,
                                int64_t ldq, const void* v, int64_t ldv, const void* out, const void* lse,
                                const void* dout, const void* bias, void* dq, void* dk_out, void* dv_out,
                                float* delta_ws, cudaStream_t st) {
  TcBwdArgs a{};
  a.S = S, a.s_real = s_real, a.H = H, a.dk = dk, a.dv = dv, a.ldq = ldq, a.ldv = ldv;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<const __nv_bfloat16*>(out);
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.bias = static_cast<const float*>(bias);
  a.lse = static_cast<const float*>(lse);
  a.dq = static_cast<__nv_bfloat16*>(dq);
  a.dk_out = static_cast<__nv_bfloat16*>(dk_out);
  a.dv_out = static_cast<__nv_bfloat16*>(dv_out);
  a.scale = (float)(1.0 / std::sqrt((double)dk));
  a.scale_l = (float)(1.4426950408889634 / std::sqrt((double)dk));
  a.vec = dk % 8 == 0 && dv % 8 == 0 && (ldq * 2) % 16 == 0 && (ldv * 2) % 16 == 0 &&
          (reinterpret_cast<uintptr_t>(q) % 16) == 0 && (reinterpret_cast<uintptr_t>(k) % 16) == 0 &&
          (reinterpret_cast<uintptr_t>(v) % 16) == 0 && (reinterpret_cast<uintptr_t>(dout) % 16) == 0;
  a.delta = delta_ws;  // [S*H] floats, the context's workspace
  switch ((dk + 15) / 16 * 16) {
    case 16: return launch_bwd_dv<16>(a, st);
    case 32: return launch_bwd_dv<32>(a, st);
    case 48: return launch_bwd_dv<48>(a, st);
    default: return launch_bwd_dv<64>(a, st);
  }
}

}  // namespace gte_b200

// Lane-piece helpers of the aligned sparse kernels (f32/bf16 shapes whose head
// chunk is a power-of-two number of 16-byte pieces, 16-byte aligned rows):
//
//   * a lane owns one 16-byte piece of one head of one node (VW = 16/sizeof(T)
//     elements; LPH lanes per head; LPN = pow2(H)*LPH lanes per node);
//   * bf16 dot products run on FHFMA.BF16 (fma.rn.f32.bf16: bf16 operands,
//     fp32 accumulate — exact products, no unpacking), f32 ones on FFMA2
//     (fma.rn.f32x2); value accumulation on FFMA2;
//   * Q/K/V finiteness is probed once per row on the row's own data.
#pragma once

#include "attn_sparse.cuh"

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

// acc[0..N) *= c on FMUL2 (the online-softmax rescale)
template <int N>
__device__ __forceinline__ void scale_pairs(float (&acc)[N], float c) {
  const uint64_t cc = pk(c, c);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(acc[2 * i], acc[2 * i + 1])), "l"(cc));
    upk(r, acc[2 * i], acc[2 * i + 1]);
  }
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
#ifndef GTE_BF16_AXPY_FHFMA
#define GTE_BF16_AXPY_FHFMA 1
#endif
  // acc[0..7] += w * x for the per-edge weights (p, dS) of the gather loops.
  // With GTE_BF16_AXPY_FHFMA the weight is rounded to bf16 — the precision
  // the P / dS operands have in FlashAttention-style bf16 kernels (and in
  // dense_tc.cu) — and the update runs on FHFMA.BF16 (bf16 operands, fp32
  // accumulate, no unpacking): 1 cvt + 8 FHFMA per edge instead of 8 unpack
  // + 4 FFMA2.
  __device__ __forceinline__ static void axpy_w(float w, const uint4& x, float (&acc)[8]) {
#if GTE_BF16_AXPY_FHFMA
    asm("{.reg .b16 wb, l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
        "cvt.rn.bf16.f32 wb, %8;\n\t"
        "mov.b32 {l0, h0}, %9;\n\tmov.b32 {l1, h1}, %10;\n\t"
        "mov.b32 {l2, h2}, %11;\n\tmov.b32 {l3, h3}, %12;\n\t"
        "fma.rn.f32.bf16 %0, wb, l0, %0;\n\tfma.rn.f32.bf16 %1, wb, h0, %1;\n\t"
        "fma.rn.f32.bf16 %2, wb, l1, %2;\n\tfma.rn.f32.bf16 %3, wb, h1, %3;\n\t"
        "fma.rn.f32.bf16 %4, wb, l2, %4;\n\tfma.rn.f32.bf16 %5, wb, h2, %5;\n\t"
        "fma.rn.f32.bf16 %6, wb, l3, %6;\n\tfma.rn.f32.bf16 %7, wb, h3, %7;}"
        : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3]), "+f"(acc[4]), "+f"(acc[5]), "+f"(acc[6]),
          "+f"(acc[7])
        : "f"(w), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
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

// This lane's piece of row 0 of a row-major tensor in a 64-bit register (the
// empty asm keeps the compiler from re-adding the uniform tensor base after
// the row offset): a gather is then one IMAD.WIDE.U32 (row * stride + base)
// instead of a multiply and a 64-bit add. Costs two live registers; it pays
// in the bf16 forward only (profiles/r2l: the backward passes and the f32
// kernels lose more to the 64-register allocation than they save).
__device__ __forceinline__ const char* lane_base(const char* base, uint32_t bo) {
  const char* b = base + bo;
  asm("" : "+l"(b));
  return b;
}
__device__ __forceinline__ uint4 ldg16r(const char* lane_row0, uint32_t row, uint32_t stride) {
  return __ldg(reinterpret_cast<const uint4*>(lane_row0 + (uint64_t)row * stride));
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

}  // namespace gte_b200

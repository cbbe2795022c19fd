// Shared device helpers for the sm_100a graph-attention kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gte_b200 {

constexpr int kWarp = 32;

// ---- storage type T -> accumulate type A ----
template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_acc(typename AccOf<T>::type x);
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// ---- softmax math. fp32 paths work in the log2 domain (one FFMA + ex2.approx
// per score); the fp64 conformance path keeps natural exp/log in the reference
// operation order (proj/src/attention.cpp:136-151). ----
template <typename A> struct SoftmaxMath;

template <> struct SoftmaxMath<float> {
  static constexpr float kLogScale = 1.4426950408889634f;  // log2(e)
  __device__ __forceinline__ static float ex(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  __device__ __forceinline__ static float lg(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  __device__ __forceinline__ static float neg_inf() { return __int_as_float(0xff800000); }
  // exact-rounding helpers so the same dot product is reproduced bit-for-bit
  // in different kernels (deg-1 rows rely on it)
  __device__ __forceinline__ static float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
};

template <> struct SoftmaxMath<double> {
  static constexpr double kLogScale = 1.0;
  __device__ __forceinline__ static double ex(double x) { return exp(x); }
  __device__ __forceinline__ static double lg(double x) { return log(x); }
  __device__ __forceinline__ static double neg_inf() { return __longlong_as_double(0xfff0000000000000ULL); }
  // fp64 conformance: multiply then add, no contraction, as the reference's
  // x86-64 -O3 build does.
  __device__ __forceinline__ static double fma(double a, double b, double c) { return __dadd_rn(__dmul_rn(a, b), c); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
};

// ---- head-chunk loads: one lane owns `n` (<= DHT) contiguous elements of a row ----
template <typename T, int DHT>
__device__ __forceinline__ void load_chunk(const T* __restrict__ p, int n, bool vec,
                                           typename AccOf<T>::type (&out)[DHT]) {
  using A = typename AccOf<T>::type;
  constexpr int kBytes = DHT * (int)sizeof(T);
  if (vec && (kBytes % 16) == 0) {
    constexpr int kVec = kBytes / 16;
    constexpr int kPer = 16 / (int)sizeof(T);
    const uint4* src = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int c = 0; c < kVec; ++c) {
      uint4 u = __ldg(src + c);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int t = 0; t < kPer; ++t) out[c * kPer + t] = to_acc(e[t]);
    }
  } else {
#pragma unroll
    for (int t = 0; t < DHT; ++t) out[t] = (t < n) ? to_acc(__ldg(p + t)) : A(0);
  }
}

template <typename T, int DHT>
__device__ __forceinline__ void store_chunk(T* __restrict__ p, int n, bool vec,
                                            const typename AccOf<T>::type (&in)[DHT]) {
  constexpr int kBytes = DHT * (int)sizeof(T);
  if (vec && (kBytes % 16) == 0) {
    constexpr int kVec = kBytes / 16;
    constexpr int kPer = 16 / (int)sizeof(T);
    uint4* dst = reinterpret_cast<uint4*>(p);
#pragma unroll
    for (int c = 0; c < kVec; ++c) {
      uint4 u;
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int t = 0; t < kPer; ++t) e[t] = from_acc<T>(in[c * kPer + t]);
      dst[c] = u;
    }
  } else {
#pragma unroll
    for (int t = 0; t < DHT; ++t)
      if (t < n) p[t] = from_acc<T>(in[t]);
  }
}

template <typename A, int DHT>
__device__ __forceinline__ A dot_chunk(const A (&a)[DHT], const A (&b)[DHT]) {
  using M = SoftmaxMath<A>;
  A acc = M::mul(a[0], b[0]);
#pragma unroll
  for (int t = 1; t < DHT; ++t) acc = M::fma(a[t], b[t], acc);
  return acc;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace gte_b200

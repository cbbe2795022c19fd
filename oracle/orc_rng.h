/* TEST INFRASTRUCTURE — not product code.
 *
 * Bit-exact C restatement of the three libstdc++ (GCC 13) random facilities the
 * reference hot path draws from:
 *   - std::mt19937_64 (standardised: [rand.predef], 312 words, MATRIX_A 0xb5026f5aa96619e9)
 *   - std::uniform_int_distribution<int64>::operator() on a 64-bit engine:
 *       Lemire "nearly divisionless" downscaling with a 128-bit product
 *       (/usr/include/c++/13/bits/uniform_int_dist.h:_S_nd)
 *   - std::shuffle: two-swaps-per-draw variant via __gen_two_uniform_ints
 *       (/usr/include/c++/13/bits/stl_algo.h:3719-3805)
 * Used by: reorder's heavy_edge_matching shuffle and restart picks
 * (reference proj/src/partition.cpp:111-114, 327-332) and partition_sequence
 * (proj/src/parallel.cpp:102-103).
 */
#ifndef ORC_RNG_H
#define ORC_RNG_H

#include <stdint.h>

typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

static inline void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    uint64_t p = g->mt[i - 1];
    g->mt[i] = 6364136223846793005ULL * (p ^ (p >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

static inline uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* Uniform integer in [0, range) for range >= 1, libstdc++ _S_nd<unsigned __int128>. */
static inline uint64_t orc_lemire(orc_mt64* g, uint64_t range) {
  unsigned __int128 prod = (unsigned __int128)orc_mt64_next(g) * range;
  uint64_t low = (uint64_t)prod;
  if (low < range) {
    uint64_t threshold = (0 - range) % range;
    while (low < threshold) {
      prod = (unsigned __int128)orc_mt64_next(g) * range;
      low = (uint64_t)prod;
    }
  }
  return (uint64_t)(prod >> 64);
}

/* std::uniform_int_distribution<int64_t>(a, b)(g) with b - a < 2^64 - 1. */
static inline int64_t orc_uniform_int(orc_mt64* g, int64_t a, int64_t b) {
  uint64_t urange = (uint64_t)b - (uint64_t)a;
  return (int64_t)((uint64_t)a + orc_lemire(g, urange + 1));
}

/* std::shuffle(first, first + n, g) on int64 elements (libstdc++ 13). */
static inline void orc_shuffle_i64(int64_t* first, int64_t n, orc_mt64* g) {
  if (n <= 0) return;
  const uint64_t urange = (uint64_t)n;
  if (UINT64_MAX / urange >= urange) {
    int64_t i = 1;
    if ((urange % 2) == 0) {
      int64_t j = (int64_t)orc_lemire(g, 2);
      int64_t t = first[i]; first[i] = first[j]; first[j] = t;
      ++i;
    }
    while (i != n) {
      const uint64_t b0 = (uint64_t)i + 1, b1 = b0 + 1;
      uint64_t x = orc_lemire(g, b0 * b1);  /* uniform in [0, b0*b1 - 1] */
      int64_t p0 = (int64_t)(x / b1), p1 = (int64_t)(x % b1);
      int64_t t = first[i]; first[i] = first[p0]; first[p0] = t;
      ++i;
      t = first[i]; first[i] = first[p1]; first[p1] = t;
      ++i;
    }
    return;
  }
  for (int64_t i = 1; i < n; ++i) {
    int64_t j = orc_uniform_int(g, 0, i);
    int64_t t = first[i]; first[i] = first[j]; first[j] = t;
  }
}

static inline uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

#endif

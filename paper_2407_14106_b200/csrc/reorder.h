// Host-side exact reorder (see reorder.cpp).
#pragma once
#include <cstdint>

namespace gte_b200 {
// Bit-identical to reference gte::reorder (proj/src/partition.cpp:413-433);
// caller validates k (power of two, 1 <= k <= n).
void reorder_exact(int64_t n, const int64_t* row_off, const int64_t* cols, int64_t k, uint64_t seed,
                   int64_t* forward, int64_t* inverse);
}  // namespace gte_b200

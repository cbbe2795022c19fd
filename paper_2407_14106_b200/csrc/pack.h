// Exact fast sub-block packer (see pack.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace gte_b200 {
// Same tile sequence as reference gte::pack_subblocks (proj/src/reformation.cpp:56-109)
// for validated arguments (1 <= d <= n_rows, n_cols; edges inside the cell, unique).
// out_rc: (row, col) origins, in placement order. want < 0: ceil(m / d^2).
int pack_subblocks_exact(const int64_t* er, const int64_t* ec, int64_t m, int64_t n_rows, int64_t n_cols,
                         int64_t d, std::vector<int64_t>& out_rc, int64_t want = -1);
}  // namespace gte_b200

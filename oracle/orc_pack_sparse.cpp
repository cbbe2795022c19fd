// TEST INFRASTRUCTURE — not product code. CPU oracle, see oracle.h.
//
// pack_subblocks restated over candidate origins instead of the coverage
// field, so the C3 layout (cells of 32768 x 32768) can be checked: the
// reference's greedy (/root/reference/proj/src/reformation.cpp:56-109) —
// `want` = ceil(nnz / d_b^2) tiles; each round takes, among the origins that
// overlap no placed tile, the one covering the most not-yet-covered edges,
// ties to the first origin in raster order; an all-zero round still places a
// tile at the first free origin; the loop stops early only if no free origin
// is left — computed the sparse way:
//
//   * an origin with cover > 0 contains an uncovered edge, so it is one of the
//     <= d_b^2 origins of that edge: covers live in a hash map keyed by the
//     raster index r0 * W + c0, bucketed by cover (ordered sets give the first
//     raster origin of the top bucket);
//   * placing a tile erases every origin it blocks (|dr| < d_b and |dc| < d_b)
//     and decrements the origins of the edges it covers;
//   * a round whose best cover would be 0 scans rows in raster order for the
//     first column not inside a blocked interval of the tiles near that row.
//
// Independent of the product's lazy-heap packer (csrc/pack.cpp); pinned
// against the reference's outputs (tests/golden/*.npz) and against the
// field-based restatement orc_pack_subblocks.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

extern "C" int orc_fail(int code, const char* fmt, ...);

namespace {
constexpr int kConfig = 2;
}

extern "C" int orc_pack_subblocks_sparse(int64_t m, const int64_t* er, const int64_t* ec, int64_t n_rows,
                                         int64_t n_cols, int64_t d_b, int64_t* tiles_rc, int64_t cap,
                                         int64_t* ntiles) {
  *ntiles = 0;
  if (d_b < 1) return orc_fail(kConfig, "pack_subblocks: d_b must be >= 1");
  if (d_b > n_rows || d_b > n_cols)
    return orc_fail(kConfig, "pack_subblocks: d_b %lld too large for %lldx%lld cell", (long long)d_b,
                    (long long)n_rows, (long long)n_cols);
  if (m == 0) return 0;
  for (int64_t e = 0; e < m; ++e)
    if (er[e] < 0 || er[e] >= n_rows || ec[e] < 0 || ec[e] >= n_cols)
      return orc_fail(kConfig, "pack_subblocks: edge outside cell");
  // unique edges sorted by (row, col); covered flags
  std::vector<std::pair<int64_t, int64_t>> edges(static_cast<size_t>(m));
  for (int64_t e = 0; e < m; ++e) edges[static_cast<size_t>(e)] = {er[e], ec[e]};
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  std::vector<char> covered(edges.size(), 0);
  const int64_t R = n_rows - d_b + 1, W = n_cols - d_b + 1;  // valid origins [0,R) x [0,W)
  auto key = [W](int64_t r, int64_t c) { return r * W + c; };

  std::unordered_map<int64_t, int> cover;
  cover.reserve(edges.size() * 8);
  for (const auto& [r, c] : edges)
    for (int64_t r0 = std::max<int64_t>(0, r - d_b + 1); r0 <= std::min(r, R - 1); ++r0)
      for (int64_t c0 = std::max<int64_t>(0, c - d_b + 1); c0 <= std::min(c, W - 1); ++c0) ++cover[key(r0, c0)];
  std::vector<std::set<int64_t>> bucket(static_cast<size_t>(d_b * d_b + 1));
  for (const auto& [k, n] : cover) bucket[static_cast<size_t>(n)].insert(k);

  const int64_t want = (m + d_b * d_b - 1) / (d_b * d_b);
  std::vector<std::pair<int64_t, int64_t>> tiles;
  auto first_free_origin = [&](int64_t* br, int64_t* bc) {
    std::vector<std::pair<int64_t, int64_t>> iv;
    for (int64_t r0 = 0; r0 < R; ++r0) {
      iv.clear();
      for (const auto& t : tiles)
        if (std::llabs(r0 - t.first) < d_b) iv.emplace_back(t.second - d_b + 1, t.second + d_b - 1);
      std::sort(iv.begin(), iv.end());
      int64_t c0 = 0;
      for (const auto& [lo, hi] : iv) {
        if (lo > c0) break;
        c0 = std::max(c0, hi + 1);
      }
      if (c0 < W) {
        *br = r0;
        *bc = c0;
        return true;
      }
    }
    return false;
  };

  while (static_cast<int64_t>(tiles.size()) < want) {
    int64_t br = -1, bc = -1;
    for (int64_t b = d_b * d_b; b >= 1; --b) {
      if (!bucket[static_cast<size_t>(b)].empty()) {
        const int64_t k = *bucket[static_cast<size_t>(b)].begin();
        br = k / W;
        bc = k % W;
        break;
      }
    }
    if (br < 0 && !first_free_origin(&br, &bc)) break;  // no free origin left
    if (static_cast<int64_t>(tiles.size()) >= cap) return orc_fail(kConfig, "pack_subblocks: tile capacity");
    tiles.emplace_back(br, bc);
    // origins blocked by the new tile leave the structure for good
    for (int64_t r0 = std::max<int64_t>(0, br - d_b + 1); r0 <= std::min(br + d_b - 1, R - 1); ++r0)
      for (int64_t c0 = std::max<int64_t>(0, bc - d_b + 1); c0 <= std::min(bc + d_b - 1, W - 1); ++c0) {
        auto it = cover.find(key(r0, c0));
        if (it == cover.end()) continue;
        bucket[static_cast<size_t>(it->second)].erase(it->first);
        cover.erase(it);
      }
    // edges inside the tile become covered: their remaining origins lose one
    for (int64_t r = br; r < br + d_b; ++r) {
      auto lo = std::lower_bound(edges.begin(), edges.end(), std::make_pair(r, bc));
      for (auto it = lo; it != edges.end() && it->first == r && it->second < bc + d_b; ++it) {
        const size_t e = static_cast<size_t>(it - edges.begin());
        if (covered[e]) continue;
        covered[e] = 1;
        const int64_t c = it->second;
        for (int64_t r0 = std::max<int64_t>(0, r - d_b + 1); r0 <= std::min(r, R - 1); ++r0)
          for (int64_t c0 = std::max<int64_t>(0, c - d_b + 1); c0 <= std::min(c, W - 1); ++c0) {
            auto f = cover.find(key(r0, c0));
            if (f == cover.end()) continue;
            bucket[static_cast<size_t>(f->second)].erase(f->first);
            if (--f->second > 0)
              bucket[static_cast<size_t>(f->second)].insert(f->first);
            else
              cover.erase(f);
          }
      }
    }
  }
  for (size_t t = 0; t < tiles.size(); ++t) {
    tiles_rc[2 * t] = tiles[t].first;
    tiles_rc[2 * t + 1] = tiles[t].second;
  }
  *ntiles = static_cast<int64_t>(tiles.size());
  return 0;
}

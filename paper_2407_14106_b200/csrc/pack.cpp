// Exact fast sub-block packer for Elastic Computation Reformation.
//
// Reference: pack_subblocks, proj/src/reformation.cpp:56-109. The reference
// rebuilds a 2-D prefix sum of the whole cell (rows x cols, 12 B per cell
// entry) and rescans every origin for every tile — at the S=256K configs a
// cell is 32768^2 and the scan is infeasible. The greedy decision it makes is
//     argmax over free origins of (cover, then smallest raster index),
//     falling back to the first free origin in raster order when no free
//     origin covers an uncovered edge, stopping when no free origin remains,
// where "free" = no overlap with an already placed tile. Here the same argmax is
// answered by a lazy max-heap over the origins that cover >= 1 uncovered edge
// (at most d_b^2 per edge), with covers decremented in place as tiles cover
// edges, and the zero-cover fallback found by a row-by-row interval scan —
// identical tile sequences at O(nnz * d_b^2 * log) instead of O(tiles * area).
#include <algorithm>
#include <cstdint>
#include <queue>
#include <unordered_map>
#include <vector>

#include "pack.h"

namespace gte_b200 {

namespace {

struct Tile {
  int64_t r, c;
};

bool overlaps(const std::vector<Tile>& tiles, int64_t r, int64_t c, int64_t d) {
  for (const Tile& t : tiles)
    if (std::llabs(r - t.r) < d && std::llabs(c - t.c) < d) return true;
  return false;
}

// Spatial hash of placed tiles on a d x d grid of buckets: an origin can only
// overlap tiles whose origin lies within d in both coordinates, i.e. in the
// 3x3 neighbourhood of its bucket.
struct TileIndex {
  int64_t d;
  std::unordered_map<uint64_t, std::vector<Tile>> buckets;
  static uint64_t key(int64_t br, int64_t bc) { return (uint64_t)br * 0x9E3779B97F4A7C15ULL ^ (uint64_t)bc; }
  void add(const Tile& t) { buckets[key(t.r / d, t.c / d)].push_back(t); }
  bool clash(int64_t r, int64_t c) const {
    const int64_t br = r / d, bc = c / d;
    for (int64_t i = br - 1; i <= br + 1; ++i)
      for (int64_t j = bc - 1; j <= bc + 1; ++j) {
        if (i < 0 || j < 0) continue;
        auto it = buckets.find(key(i, j));
        if (it == buckets.end()) continue;
        for (const Tile& t : it->second)
          if (std::llabs(r - t.r) < d && std::llabs(c - t.c) < d) return true;
      }
    return false;
  }
};

}  // namespace

int pack_subblocks_exact(const int64_t* er, const int64_t* ec, int64_t m, int64_t n_rows, int64_t n_cols,
                         int64_t d, std::vector<int64_t>& out_rc, int64_t want) {
  out_rc.clear();
  if (m == 0) return 0;
  if (want < 0) want = (m + d * d - 1) / (d * d);
  const int64_t R = n_rows - d, Cc = n_cols - d;  // origin ranges [0, R] x [0, Cc]
  const int64_t W = Cc + 1;                         // raster stride of origins

  // cover of every origin touching >= 1 edge
  std::vector<int64_t> keys;
  keys.reserve((size_t)m * (size_t)std::min<int64_t>(d * d, 1 << 20));
  for (int64_t e = 0; e < m; ++e) {
    const int64_t r0 = std::max<int64_t>(0, er[e] - d + 1), r1 = std::min(er[e], R);
    const int64_t c0 = std::max<int64_t>(0, ec[e] - d + 1), c1 = std::min(ec[e], Cc);
    for (int64_t r = r0; r <= r1; ++r)
      for (int64_t c = c0; c <= c1; ++c) keys.push_back(r * W + c);
  }
  std::sort(keys.begin(), keys.end());
  std::vector<int64_t> cand;    // distinct origin raster ids, ascending
  std::vector<int64_t> cover;   // current cover per candidate
  cand.reserve(keys.size() / 2 + 1);
  for (size_t i = 0; i < keys.size();) {
    size_t j = i;
    while (j < keys.size() && keys[j] == keys[i]) ++j;
    cand.push_back(keys[i]);
    cover.push_back((int64_t)(j - i));
    i = j;
  }
  keys.clear();
  keys.shrink_to_fit();
  auto find = [&](int64_t id) -> int64_t {
    auto it = std::lower_bound(cand.begin(), cand.end(), id);
    return (it != cand.end() && *it == id) ? (int64_t)(it - cand.begin()) : -1;
  };

  // uncovered edges by cell coordinate, for zeroing a placed tile
  std::unordered_map<int64_t, int> edge_at;
  edge_at.reserve((size_t)m * 2);
  for (int64_t e = 0; e < m; ++e) edge_at[er[e] * n_cols + ec[e]] = 1;

  struct HE {
    int64_t cover, id;
    bool operator<(const HE& o) const { return cover != o.cover ? cover < o.cover : id > o.id; }
  };
  std::priority_queue<HE> heap;
  for (size_t i = 0; i < cand.size(); ++i) heap.push({cover[i], cand[i]});

  std::vector<Tile> tiles;
  TileIndex index{d, {}};
  while ((int64_t)tiles.size() < want) {
    int64_t pick = -1;
    while (!heap.empty()) {
      HE t = heap.top();
      const int64_t ci = find(t.id);
      if (cover[ci] != t.cover || t.cover <= 0) {
        heap.pop();
        continue;
      }
      if (index.clash(t.id / W, t.id % W)) {
        heap.pop();  // blocked forever
        continue;
      }
      pick = t.id;
      heap.pop();
      break;
    }
    Tile chosen;
    if (pick >= 0) {
      chosen = {pick / W, pick % W};
    } else {
      // no free origin covers an uncovered edge: first free origin in raster order
      bool found = false;
      for (int64_t r = 0; r <= R && !found; ++r) {
        std::vector<std::pair<int64_t, int64_t>> blocked;
        for (const Tile& t : tiles)
          if (std::llabs(r - t.r) < d) blocked.emplace_back(t.c - d + 1, t.c + d - 1);
        std::sort(blocked.begin(), blocked.end());
        int64_t c = 0;
        for (auto& [lo, hi] : blocked) {
          if (c < lo) break;
          if (c <= hi) c = hi + 1;
        }
        if (c <= Cc) {
          chosen = {r, c};
          found = true;
        }
      }
      if (!found) break;
    }
    tiles.push_back(chosen);
    index.add(chosen);
    // zero the covered edges; decrement the covers of every origin seeing them
    for (int64_t r = chosen.r; r < chosen.r + d; ++r)
      for (int64_t c = chosen.c; c < chosen.c + d; ++c) {
        auto it = edge_at.find(r * n_cols + c);
        if (it == edge_at.end() || it->second == 0) continue;
        it->second = 0;
        const int64_t r0 = std::max<int64_t>(0, r - d + 1), r1 = std::min(r, R);
        const int64_t c0 = std::max<int64_t>(0, c - d + 1), c1 = std::min(c, Cc);
        for (int64_t orr = r0; orr <= r1; ++orr)
          for (int64_t occ = c0; occ <= c1; ++occ) {
            const int64_t id = orr * W + occ;
            const int64_t ci = find(id);
            if (--cover[ci] > 0) heap.push({cover[ci], id});
          }
      }
  }
  out_rc.reserve(tiles.size() * 2);
  for (const Tile& t : tiles) {
    out_rc.push_back(t.r);
    out_rc.push_back(t.c);
  }
  (void)overlaps;
  return 0;
}

}  // namespace gte_b200

// Community-ordered execution schedule for the sparse attention kernels.
//
// The reference's cluster-aware reorder (proj/src/partition.cpp:413-433) cuts
// the sequence into k (= 8 at C3) clusters of S/k positions; inside a cluster
// positions keep the input order, so the K/V rows one row gathers are spread
// over the whole cluster (16 MB at S = 256K, f32) and an SM's L1 sees almost
// no reuse (3% of gathers repeat inside a 128-row window, measured on C3).
// Executing rows in *community* order instead — rows whose neighbourhoods
// overlap processed back to back by the same CTA — lets L1 serve most of the
// gathers (71% repeats inside a 128-row window).
//
// This is an execution order only: every row is still computed by one slot
// with the same arithmetic, outputs are written at the row's own position,
// so results are bit-identical with or without it. It is built once per
// pattern (like the CSC view) by synchronous label propagation over the
// symmetrised pattern: every node takes the most frequent label among its
// neighbours (ties -> smallest label), all nodes at once from the previous
// round's labels (deterministic, thread-count independent), until < 0.1% of
// labels change or `iters` rounds. Rows are then ordered by (label, row).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
}
using gte_b200::set_error;

namespace {

template <typename F>
void parallel_for(int64_t n, F&& f) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 32) nt = 32;
  if (n < 65536) nt = 1;
  if (nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t a = t * per, b = std::min<int64_t>(n, a + per);
    if (a >= b) break;
    th.emplace_back([&f, a, b] { f(a, b); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int gte_community_order(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t iters,
                        int64_t* order, int64_t* n_communities) {
  if (n < 0 || nnz < 0) return set_error(GTE_CONFIG, "schedule: negative size");
  if (n == 0) {
    if (n_communities) *n_communities = 0;
    return GTE_OK;
  }
  if (row_off[0] != 0 || row_off[n] != nnz) return set_error(GTE_CONFIG, "schedule: malformed offsets");
  // symmetrised adjacency without self-loops: out-arcs then in-arcs per node
  std::vector<int64_t> deg(n + 1, 0);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const int64_t v = cols[e];
      if (v < 0 || v >= n) return set_error(GTE_CONFIG, "schedule: column out of range");
      if (v == u) continue;
      ++deg[u + 1];
      ++deg[v + 1];
    }
  for (int64_t u = 0; u < n; ++u) deg[u + 1] += deg[u];
  std::vector<int32_t> adj(deg[n] > 0 ? deg[n] : 1);
  {
    std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
    for (int64_t u = 0; u < n; ++u)
      for (int64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
        const int64_t v = cols[e];
        if (v == u) continue;
        adj[fill[u]++] = (int32_t)v;
        adj[fill[v]++] = (int32_t)u;
      }
  }
  std::vector<int32_t> lab(n), nxt(n);
  for (int64_t u = 0; u < n; ++u) lab[u] = (int32_t)u;
  for (int64_t it = 0; it < iters; ++it) {
    std::atomic_int64_t changed{0};
    parallel_for(n, [&](int64_t a, int64_t b) {
      std::vector<int32_t> buf;
      int64_t ch = 0;
      for (int64_t u = a; u < b; ++u) {
        const int64_t d0 = deg[u], d1 = deg[u + 1];
        if (d0 == d1) {
          nxt[u] = lab[u];
          continue;
        }
        buf.resize(d1 - d0);
        for (int64_t e = d0; e < d1; ++e) buf[e - d0] = lab[adj[e]];
        std::sort(buf.begin(), buf.end());
        int32_t best = buf[0];
        int64_t best_n = 0;
        for (size_t s = 0; s < buf.size();) {
          size_t t = s;
          while (t < buf.size() && buf[t] == buf[s]) ++t;
          if ((int64_t)(t - s) > best_n) {
            best_n = (int64_t)(t - s);
            best = buf[s];
          }
          s = t;
        }
        nxt[u] = best;
        ch += best != lab[u];
      }
      changed += ch;
    });
    lab.swap(nxt);
    if (changed.load() * 1000 < n) break;
  }
  // order by (label, row): counting sort over labels
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t u = 0; u < n; ++u) ++cnt[lab[u] + 1];
  int64_t comms = 0;
  for (int64_t l = 0; l < n; ++l) {
    comms += cnt[l + 1] > 0;
    cnt[l + 1] += cnt[l];
  }
  for (int64_t u = 0; u < n; ++u) order[cnt[lab[u]]++] = u;
  if (n_communities) *n_communities = comms;
  return GTE_OK;
}

}  // extern "C"

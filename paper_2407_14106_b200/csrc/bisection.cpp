// Host half of the cluster-aware reorder (bisection.h): the greedy passes
// whose decision order the reference fixes (proj/src/partition.cpp), each
// answered with a priority queue instead of a full scan per decision, and a
// driver that hands every level's graph transforms to the GPU
// (partition_gpu.cu) and runs the two halves of each bisection concurrently.
//
// Decision rules (all ties to the smallest node id):
//   matching     nodes visited in std::shuffle order; an unmatched node takes
//                its heaviest unmatched neighbour (:111-138)
//   coarsening   until <= 64 nodes or a level keeps > 95 % of them (:315-321)
//   seeds        4 trials: pseudo-peripheral node (two BFS sweeps, farthest =
//                deepest) or a random one, grown to half the weight by
//                strongest connection, FM-refined, best cut kept (:326-339)
//   FM           repeatedly move the unlocked node of highest gain whose move
//                keeps |w0 - w1| <= allowance, then roll back to the best
//                prefix; up to 10 passes while a pass gains (:187-245)
//   rebalance    move the best-gain node of the heavy side that does not
//                overshoot until |w0 - w1| <= 1 (:281-305)
// Random draws are libstdc++'s std::mt19937_64 / std::shuffle /
// std::uniform_int_distribution, the reference's, in the same order.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <numeric>
#include <queue>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>
#include <chrono>
#include <cstdio>
#include <mutex>

#include "bisection.h"

namespace gte_b200 {
namespace part {
namespace {

// GTE_REORDER_TRACE=1: per-phase wall time on stderr (profiling only)
struct Trace {
  bool on = getenv("GTE_REORDER_TRACE") != nullptr;
  std::mutex mu;
  double t[8] = {};
  static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
  void add(int i, double dt) {
    if (!on) return;
    std::lock_guard<std::mutex> l(mu);
    t[i] += dt;
  }
};
Trace& trace() {
  static Trace tr;
  return tr;
}

constexpr int kFmPassLimit = 10;        // partition.cpp:17
constexpr double kImbalanceTol = 0.05;  // partition.cpp:18
constexpr int64_t kCoarseStop = 64;     // partition.cpp:315
constexpr double kMinShrink = 0.95;     // partition.cpp:319
constexpr int kSeedTrials = 4;          // partition.cpp:326
constexpr int64_t kParallelNodes = 8192;  // halves below this size recurse inline

uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kSaltRoot = 0xda3e39cb94b95bdbULL, kSaltLo = 0x517cc1b727220a95ULL,
                   kSaltHi = 0x2545f4914f6cdd1dULL;

// Lazy max-queue of (key, node): highest key first, then the smallest node.
// Stale entries are skipped by the caller's validity test.
class MaxQueue {
 public:
  void push(int64_t key, int32_t v) { q_.push(Item{key, v}); }
  template <typename Valid>
  bool top(Valid&& valid, int64_t* key, int32_t* v) {
    while (!q_.empty()) {
      const Item& t = q_.top();
      if (valid(t.key, t.v)) {
        *key = t.key;
        *v = t.v;
        return true;
      }
      q_.pop();
    }
    return false;
  }
  void clear() { q_ = decltype(q_)(); }

 private:
  struct Item {
    int64_t key;
    int32_t v;
    bool operator<(const Item& o) const { return key != o.key ? key < o.key : v > o.v; }
  };
  std::priority_queue<Item> q_;
};

int64_t weight_of(const WGraph& g) {
  int64_t s = 0;
  for (int32_t w : g.vw) s += w;
  return s;
}

// partition.cpp:168-184: cut weight; allowance = max(2 * tol * W, 2 * heaviest node)
int64_t cut_of(const WGraph& g, const std::vector<uint8_t>& side) {
  int64_t twice = 0;
  for (int64_t u = 0; u < g.n; ++u)
    for (int64_t a = g.xoff[u]; a < g.xoff[u + 1]; ++a)
      if (side[u] != side[g.nbr[a]]) twice += g.wt[a];
  return twice / 2;
}
int64_t allowance_of(const WGraph& g) {
  int64_t heaviest = 1;
  if (g.n) heaviest = *std::max_element(g.vw.begin(), g.vw.end());
  const auto tol = static_cast<int64_t>(2 * kImbalanceTol * static_cast<double>(weight_of(g)));
  return tol > 2 * heaviest ? tol : 2 * heaviest;
}

std::vector<int32_t> heavy_matching(const WGraph& g, std::mt19937_64& rng) {
  std::vector<int32_t> visit(g.n);
  std::iota(visit.begin(), visit.end(), 0);
  std::shuffle(visit.begin(), visit.end(), rng);
  std::vector<int32_t> mate(g.n, -1);
  for (int32_t u : visit) {
    if (mate[u] >= 0) continue;
    int32_t take = -1, take_w = 0;
    for (int64_t a = g.xoff[u]; a < g.xoff[u + 1]; ++a) {
      const int32_t v = g.nbr[a];
      if (mate[v] >= 0) continue;
      if (take < 0 || g.wt[a] > take_w || (g.wt[a] == take_w && v < take)) {
        take = v;
        take_w = g.wt[a];
      }
    }
    if (take >= 0) {
      mate[u] = take;
      mate[take] = u;
    }
  }
  for (int64_t u = 0; u < g.n; ++u)
    if (mate[u] < 0) mate[u] = (int32_t)u;
  return mate;
}

// deepest node reached from src (BFS), smallest id among the deepest
int32_t deepest_from(const WGraph& g, int32_t src, std::vector<int32_t>& depth, std::vector<int32_t>& queue) {
  std::fill(depth.begin(), depth.end(), -1);
  queue.clear();
  queue.push_back(src);
  depth[src] = 0;
  for (size_t h = 0; h < queue.size(); ++h) {
    const int32_t u = queue[h];
    for (int64_t a = g.xoff[u]; a < g.xoff[u + 1]; ++a)
      if (depth[g.nbr[a]] < 0) {
        depth[g.nbr[a]] = depth[u] + 1;
        queue.push_back(g.nbr[a]);
      }
  }
  int32_t best = src;
  for (int64_t v = 0; v < g.n; ++v)
    if (depth[v] > depth[best] || (depth[v] == depth[best] && v < best)) best = (int32_t)v;
  return best;
}

// side 0 grows from `seed` by strongest connection until it holds half the weight
std::vector<uint8_t> grow_half(const WGraph& g, int32_t seed) {
  std::vector<uint8_t> side(g.n, 1);
  std::vector<int64_t> link(g.n, 0);
  MaxQueue q;
  for (int64_t v = 0; v < g.n; ++v) q.push(0, (int32_t)v);
  const int64_t half = weight_of(g) / 2;
  int64_t held = 0, taken = 0;
  int32_t next = seed;
  for (;;) {
    side[next] = 0;
    held += g.vw[next];
    ++taken;
    for (int64_t a = g.xoff[next]; a < g.xoff[next + 1]; ++a) {
      const int32_t v = g.nbr[a];
      if (!side[v]) continue;
      link[v] += g.wt[a];
      q.push(link[v], v);
    }
    if (held >= half || taken == g.n) break;
    int64_t key;
    int32_t v;
    if (!q.top([&](int64_t k, int32_t x) { return side[x] && link[x] == k; }, &key, &v)) break;
    next = v;
  }
  return side;
}

// Distinct node weights, ascending; a move of weight w from side s is
// feasible iff |D_s - 2w| <= allow (D_s = W_s - W_other), a contiguous range
// of classes, scanned from the light end.
struct WeightClasses {
  std::vector<int64_t> w;
  std::vector<int32_t> of;
  explicit WeightClasses(const WGraph& g) {
    w.assign(g.vw.begin(), g.vw.end());
    std::sort(w.begin(), w.end());
    w.erase(std::unique(w.begin(), w.end()), w.end());
    of.resize(g.n);
    for (int64_t v = 0; v < g.n; ++v) of[v] = (int32_t)(std::lower_bound(w.begin(), w.end(), g.vw[v]) - w.begin());
  }
};

// Best (key desc, node asc) over a range of weight classes: a tournament
// tree whose leaf c holds the best entry pushed into class c since its last
// refresh. A leaf entry that is still valid is its class's best valid node
// (every node in the class queue is either older, hence no better than the
// refreshed top, or a later push, hence no better than the leaf); an invalid
// one is refreshed from the class queue. One range query per FM decision
// instead of a scan over every feasible class.
class ClassTournament {
 public:
  void reset(size_t n) {
    size_ = 1;
    while (size_ < n) size_ <<= 1;
    key_.assign(2 * size_, kNoKey);
    id_.assign(2 * size_, kNoId);
  }
  void offer(size_t c, int64_t key, int32_t id) {  // a push into class c
    size_t x = size_ + c;
    if (!better(key, id, key_[x], id_[x])) return;
    key_[x] = key;
    id_[x] = id;
    for (x >>= 1; x; x >>= 1) pull(x);
  }
  void set(size_t c, int64_t key, int32_t id) {  // refreshed leaf
    size_t x = size_ + c;
    key_[x] = key;
    id_[x] = id;
    for (x >>= 1; x; x >>= 1) pull(x);
  }
  // class index of the best leaf in [lo, hi], or -1 when all are empty
  long best(size_t lo, size_t hi, int64_t* key, int32_t* id) const {
    long at = -1;
    int64_t bk = kNoKey;
    int32_t bi = kNoId;
    auto take = [&](size_t x) {
      // descend to the leaf that holds node x's winner
      if (!better(key_[x], id_[x], bk, bi)) return;
      while (x < size_) x = (key_[2 * x] == key_[x] && id_[2 * x] == id_[x]) ? 2 * x : 2 * x + 1;
      at = (long)(x - size_);
      bk = key_[x];
      bi = id_[x];
    };
    for (size_t l = lo + size_, r = hi + size_ + 1; l < r; l >>= 1, r >>= 1) {
      if (l & 1) take(l++);
      if (r & 1) take(--r);
    }
    *key = bk;
    *id = bi;
    return bk == kNoKey && bi == kNoId ? -1 : at;
  }

 private:
  static constexpr int64_t kNoKey = INT64_MIN;
  static constexpr int32_t kNoId = INT32_MAX;
  static bool better(int64_t k1, int32_t i1, int64_t k2, int32_t i2) { return k1 != k2 ? k1 > k2 : i1 < i2; }
  void pull(size_t x) {
    const size_t w = better(key_[2 * x], id_[2 * x], key_[2 * x + 1], id_[2 * x + 1]) ? 2 * x : 2 * x + 1;
    key_[x] = key_[w];
    id_[x] = id_[w];
  }
  size_t size_ = 1;
  std::vector<int64_t> key_;
  std::vector<int32_t> id_;
};

class FmRefiner {
 public:
  FmRefiner(const WGraph& g, std::vector<uint8_t>& side, int64_t allow)
      : g_(g), side_(side), allow_(allow), cls_(g), gain_(g.n), locked_(g.n), queues_(2 * cls_.w.size()) {}

  void run() {
    for (int pass = 0; pass < kFmPassLimit; ++pass)
      if (!one_pass()) break;
  }

 private:
  MaxQueue& queue(int s, int c) { return queues_[s * cls_.w.size() + c]; }
  void push(int s, int c, int64_t key, int32_t v) {
    queue(s, c).push(key, v);
    tour_[s].offer((size_t)c, key, v);
  }

  bool one_pass() {
    load_[0] = load_[1] = 0;
    for (int64_t v = 0; v < g_.n; ++v) load_[side_[v]] += g_.vw[v];
    for (auto& q : queues_) q.clear();
    tour_[0].reset(cls_.w.size());
    tour_[1].reset(cls_.w.size());
    for (int64_t v = 0; v < g_.n; ++v) {
      int64_t s = 0;
      for (int64_t a = g_.xoff[v]; a < g_.xoff[v + 1]; ++a) s += side_[g_.nbr[a]] != side_[v] ? g_.wt[a] : -g_.wt[a];
      gain_[v] = s;
      locked_[v] = 0;
      push(side_[v], cls_.of[v], s, (int32_t)v);
    }
    std::vector<int32_t> order;
    order.reserve(g_.n);
    int64_t run = 0, best = 0;
    size_t keep = 0;
    int32_t v;
    while ((v = pick()) >= 0) {
      move(v);
      locked_[v] = 1;
      run += gain_[v];
      order.push_back(v);
      for (int64_t a = g_.xoff[v]; a < g_.xoff[v + 1]; ++a) {
        const int32_t x = g_.nbr[a];
        if (locked_[x]) continue;
        gain_[x] += side_[x] == side_[v] ? -2 * (int64_t)g_.wt[a] : 2 * (int64_t)g_.wt[a];
        push(side_[x], cls_.of[x], gain_[x], x);
      }
      if (run > best) {
        best = run;
        keep = order.size();
      }
    }
    while (order.size() > keep) {  // undo the moves after the best prefix
      move(order.back());
      order.pop_back();
    }
    return best > 0;
  }

  // best feasible unlocked node over both sides and all feasible classes:
  // a move of weight w from side s is feasible iff -allow <= D_s - 2w <= allow
  int32_t pick() {
    int32_t who = -1;
    int64_t who_gain = 0;
    const size_t nc = cls_.w.size();
    for (int s = 0; s < 2; ++s) {
      const int64_t d = load_[s] - load_[1 - s];
      // classes ascending by weight: D - 2w decreases; feasible = [lo, hi]
      size_t lo = 0, hi = nc;
      {
        size_t a = 0, b = nc;  // first c with d - 2w <= allow
        while (a < b) {
          const size_t m = (a + b) / 2;
          if (d - 2 * cls_.w[m] <= allow_) b = m; else a = m + 1;
        }
        lo = a;
        a = lo, b = nc;  // first c with d - 2w < -allow
        while (a < b) {
          const size_t m = (a + b) / 2;
          if (d - 2 * cls_.w[m] < -allow_) b = m; else a = m + 1;
        }
        hi = a;  // exclusive
      }
      if (lo >= hi) continue;
      auto ok = [&](int64_t k, int32_t y) { return !locked_[y] && side_[y] == s && gain_[y] == k; };
      for (;;) {
        int64_t key;
        int32_t x;
        const long c = tour_[s].best(lo, hi - 1, &key, &x);
        if (c < 0) break;
        if (ok(key, x)) {
          if (who < 0 || key > who_gain || (key == who_gain && x < who)) {
            who = x;
            who_gain = key;
          }
          break;
        }
        // stale leaf: refresh it from its class queue
        int64_t tk;
        int32_t tx;
        if (queue(s, (int)c).top(ok, &tk, &tx)) tour_[s].set((size_t)c, tk, tx);
        else tour_[s].set((size_t)c, INT64_MIN, INT32_MAX);
      }
    }
    return who;
  }

  void move(int32_t v) {
    const int s = side_[v];
    side_[v] = (uint8_t)(1 - s);
    load_[s] -= g_.vw[v];
    load_[1 - s] += g_.vw[v];
  }

  const WGraph& g_;
  std::vector<uint8_t>& side_;
  int64_t allow_;
  WeightClasses cls_;
  std::vector<int64_t> gain_;
  std::vector<uint8_t> locked_;
  std::vector<MaxQueue> queues_;
  ClassTournament tour_[2];
  int64_t load_[2] = {0, 0};
};

// heavy side gives up its best-gain nodes (no overshoot) until |w0 - w1| <= 1
void rebalance(const WGraph& g, std::vector<uint8_t>& side) {
  int64_t load[2] = {0, 0};
  for (int64_t v = 0; v < g.n; ++v) load[side[v]] += g.vw[v];
  if (std::llabs(load[0] - load[1]) <= 1) return;
  const int heavy = load[0] > load[1] ? 0 : 1;
  WeightClasses cls(g);
  std::vector<int64_t> gain(g.n, 0);
  std::vector<MaxQueue> q(cls.w.size());
  for (int64_t v = 0; v < g.n; ++v) {
    if (side[v] != heavy) continue;
    int64_t s = 0;
    for (int64_t a = g.xoff[v]; a < g.xoff[v + 1]; ++a) s += side[g.nbr[a]] != heavy ? g.wt[a] : -g.wt[a];
    gain[v] = s;
    q[cls.of[v]].push(s, (int32_t)v);
  }
  // a move never overshoots, so the heavy side stays heavy
  while (load[heavy] - load[1 - heavy] > 1) {
    const int64_t excess = load[heavy] - load[1 - heavy];
    int32_t who = -1;
    int64_t who_gain = 0;
    for (size_t c = 0; c < cls.w.size() && 2 * cls.w[c] <= excess; ++c) {
      int64_t key;
      int32_t x;
      if (!q[c].top([&](int64_t k, int32_t y) { return side[y] == heavy && gain[y] == k; }, &key, &x)) continue;
      if (who < 0 || key > who_gain || (key == who_gain && x < who)) {
        who = x;
        who_gain = key;
      }
    }
    if (who < 0) break;
    side[who] = (uint8_t)(1 - heavy);
    load[heavy] -= g.vw[who];
    load[1 - heavy] += g.vw[who];
    for (int64_t a = g.xoff[who]; a < g.xoff[who + 1]; ++a) {
      const int32_t x = g.nbr[a];
      if (side[x] != heavy) continue;
      gain[x] += 2 * (int64_t)g.wt[a];
      q[cls.of[x]].push(gain[x], x);
    }
  }
}

// one bisection (partition.cpp:310-350): coarsen, seed, project + refine
std::vector<uint8_t> bisect_level(cudaStream_t st, const WGraph& g, std::mt19937_64& rng) {
  if (g.n == 1) return {0};
  std::vector<WGraph> coarse;  // coarse[l] = level l + 1
  std::vector<std::vector<int32_t>> maps;
  const WGraph* cur = &g;
  while (cur->n > kCoarseStop) {
    double t0 = Trace::now();
    const std::vector<int32_t> mate = heavy_matching(*cur, rng);
    double t1 = Trace::now();
    WGraph c;
    std::vector<int32_t> cmap;
    dev_contract(st, *cur, mate, c, cmap);
    trace().add(0, t1 - t0);
    trace().add(1, Trace::now() - t1);
    if (static_cast<double>(c.n) > kMinShrink * static_cast<double>(cur->n)) break;
    maps.push_back(std::move(cmap));
    coarse.push_back(std::move(c));
    cur = &coarse.back();
  }
  const WGraph& top = *cur;
  std::uniform_int_distribution<int64_t> any(0, top.n - 1);
  std::vector<int32_t> depth(top.n), queue;
  std::vector<uint8_t> side;
  int64_t best_cut = -1;
  for (int t = 0; t < kSeedTrials; ++t) {
    const int32_t far1 = deepest_from(top, (int32_t)any(rng), depth, queue);
    const int32_t far2 = deepest_from(top, far1, depth, queue);
    std::vector<uint8_t> trial = grow_half(top, t == 0 ? far2 : (int32_t)any(rng));
    FmRefiner(top, trial, allowance_of(top)).run();
    const int64_t c = cut_of(top, trial);
    if (best_cut < 0 || c < best_cut) {
      best_cut = c;
      side = std::move(trial);
    }
  }
  for (size_t l = maps.size(); l-- > 0;) {  // project onto level l and refine there
    const WGraph& fine = l == 0 ? g : coarse[l - 1];
    std::vector<uint8_t> f(fine.n);
    for (int64_t v = 0; v < fine.n; ++v) f[v] = side[maps[l][v]];
    side = std::move(f);
    const double t0 = Trace::now();
    FmRefiner(fine, side, allowance_of(fine)).run();
    trace().add(l == 0 ? 2 : 3, Trace::now() - t0);
  }
  const double t0 = Trace::now();
  rebalance(g, side);
  const double t1 = Trace::now();
  FmRefiner(g, side, 1).run();
  trace().add(4, t1 - t0);
  trace().add(5, Trace::now() - t1);
  return side;
}

struct Worker {
  cudaStream_t st = nullptr;
  Worker() {
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      throw std::runtime_error("reorder: cannot create a CUDA stream");
  }
  ~Worker() { cudaStreamDestroy(st); }
};

// partition.cpp:352-391: parts [base, base + k) for the nodes `ids` of g
void split_into(const WGraph& g, const std::vector<int32_t>& ids, int64_t k, uint64_t seed, int64_t base,
                std::vector<int64_t>& part, int device) {
  if (k == 1 || g.n == 0) {
    for (int32_t v : ids) part[v] = base;
    return;
  }
  cudaSetDevice(device);
  Worker w;
  std::mt19937_64 rng(mix64(seed));
  std::vector<uint8_t> side = bisect_level(w.st, g, rng);
  WGraph sub[2];
  std::vector<int32_t> local[2];
  const double ts = Trace::now();
  dev_split(w.st, g, side, sub, local);
  trace().add(6, Trace::now() - ts);
  std::vector<int32_t> sub_ids[2];
  for (int s = 0; s < 2; ++s) {
    sub_ids[s].resize(local[s].size());
    for (size_t i = 0; i < local[s].size(); ++i) sub_ids[s][i] = ids[local[s][i]];
  }
  const uint64_t s0 = mix64(seed ^ kSaltLo), s1 = mix64(seed ^ kSaltHi);
  if (sub[0].n >= kParallelNodes && sub[1].n >= kParallelNodes) {
    std::exception_ptr err;
    std::thread t([&] {
      try {
        split_into(sub[0], sub_ids[0], k / 2, s0, base, part, device);
      } catch (...) {
        err = std::current_exception();
      }
    });
    split_into(sub[1], sub_ids[1], k / 2, s1, base + k / 2, part, device);
    t.join();
    if (err) std::rethrow_exception(err);
  } else {
    split_into(sub[0], sub_ids[0], k / 2, s0, base, part, device);
    split_into(sub[1], sub_ids[1], k / 2, s1, base + k / 2, part, device);
  }
}

}  // namespace
}  // namespace part

void reorder_cluster(int64_t n, const int64_t* row_off, const int64_t* cols, int64_t k, uint64_t seed,
                     int64_t* forward, int64_t* inverse) {
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) throw std::runtime_error("reorder: no CUDA device");
  part::WGraph g;
  {
    part::Worker w;
    part::dev_symmetrize(w.st, n, row_off, cols, g);
  }
  std::vector<int32_t> ids(n);
  std::iota(ids.begin(), ids.end(), 0);
  std::vector<int64_t> pid(n, 0);
  const double t0 = part::Trace::now();
  part::split_into(g, ids, k, part::mix64(seed ^ part::kSaltRoot), 0, pid, device);
  if (part::trace().on) {
    const double* t = part::trace().t;
    fprintf(stderr, "reorder trace: total %.2f s | match %.2f contract(dev) %.2f fm_finest %.2f fm_coarse %.2f "
            "rebalance %.2f fm_final %.2f split(dev) %.2f (thread-summed)\n", part::Trace::now() - t0, t[0], t[1], t[2],
            t[3], t[4], t[5], t[6]);
  }
  // stable order by part (partition.cpp:423-431): counting sort
  std::vector<int64_t> start(k + 1, 0);
  for (int64_t v = 0; v < n; ++v) ++start[pid[v] + 1];
  std::partial_sum(start.begin(), start.end(), start.begin());
  for (int64_t v = 0; v < n; ++v) inverse[start[pid[v]]++] = v;
  for (int64_t p = 0; p < n; ++p) forward[inverse[p]] = p;
}

}  // namespace gte_b200

// Host-side pieces of the hot path's control logic (C ABI part 3):
//   - ECR tuner + hyper-parameter model   reference proj/src/reformation.cpp:224-296
//   - interleave conditions / mode         reference proj/src/interleave.cpp:68-106
//   - sequence partition (pad + shuffle)   reference proj/src/parallel.cpp:96-113
// These are scalar or BFS control decisions taken once per epoch / per
// sequence; they run on the host in C++ (libstdc++ std::shuffle and
// std::mt19937_64 reproduce the reference's draws exactly).
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
}
using gte_b200::set_error;

struct gte_tuner {
  double avg_loss = 0.0;
  std::vector<std::pair<int64_t, double>> ldr;
  std::vector<double> thresholds;
  size_t idx = 0;
  int64_t delta = 10;
  bool has_loss = false;
};

extern "C" {

// make_tuner_state (reformation.cpp:224-238)
int gte_tuner_create(double beta_g, int64_t delta, gte_tuner** out) {
  if (beta_g < 0.0 || beta_g > 1.0) return set_error(GTE_CONFIG, "tuner: beta_g must lie in [0, 1]");
  if (delta < 1) return set_error(GTE_CONFIG, "tuner: delta must be >= 1");
  auto* st = new gte_tuner();
  st->delta = delta;
  std::vector<double> raw = {0.0, beta_g, 1.5 * beta_g, 5.0 * beta_g, 7.0 * beta_g, 10.0 * beta_g, 1.0};
  for (double& v : raw) v = std::min(v, 1.0);
  std::sort(raw.begin(), raw.end());
  raw.erase(std::unique(raw.begin(), raw.end()), raw.end());
  st->thresholds = raw;
  st->idx = (size_t)(std::lower_bound(raw.begin(), raw.end(), std::min(beta_g, 1.0)) - raw.begin());
  *out = st;
  return GTE_OK;
}

// tuner_update (reformation.cpp:240-265)
int gte_tuner_update(gte_tuner* st, double loss, double epoch_time_s, int64_t epoch) {
  if (epoch_time_s <= 0.0) return set_error(GTE_CONFIG, "tuner_update: epoch_time must be positive");
  if (!st->has_loss) {
    st->avg_loss = loss;
    st->has_loss = true;
    st->ldr.emplace_back(epoch, 0.0);
    return GTE_OK;
  }
  if (!st->ldr.empty() && epoch != st->ldr.back().first + 1)
    return set_error(GTE_CONFIG, "tuner_update: epochs must be consecutive");
  const double prev = st->avg_loss;
  st->avg_loss = 0.9 * prev + 0.1 * loss;
  const double ldr = (st->avg_loss - prev) / epoch_time_s;
  st->ldr.emplace_back(epoch, ldr);
  const int64_t lag = (int64_t)st->ldr.size() - 1 - st->delta;
  if (epoch >= st->delta && lag >= 0) {
    if (ldr >= st->ldr[(size_t)lag].second)
      st->idx = std::min(st->idx + 1, st->thresholds.size() - 1);
    else if (st->idx > 0)
      --st->idx;
  }
  return GTE_OK;
}

int gte_tuner_state(const gte_tuner* st, double* avg_loss, int64_t* idx, double* thresholds, int64_t* n_thresholds,
                    int32_t* has_loss) {
  if (avg_loss) *avg_loss = st->avg_loss;
  if (idx) *idx = (int64_t)st->idx;
  if (n_thresholds) *n_thresholds = (int64_t)st->thresholds.size();
  if (thresholds) std::copy(st->thresholds.begin(), st->thresholds.end(), thresholds);
  if (has_loss) *has_loss = st->has_loss;
  return GTE_OK;
}

int gte_tuner_history(const gte_tuner* st, int64_t* epochs, double* ldr, int64_t* n) {
  if (n) *n = (int64_t)st->ldr.size();
  for (size_t i = 0; i < st->ldr.size(); ++i) {
    if (epochs) epochs[i] = st->ldr[i].first;
    if (ldr) ldr[i] = st->ldr[i].second;
  }
  return GTE_OK;
}

int gte_tuner_set(gte_tuner* st, double avg_loss, int64_t idx, int32_t has_loss, int64_t n_hist, const int64_t* epochs,
                  const double* ldr) {
  st->avg_loss = avg_loss;
  st->idx = (size_t)idx;
  st->has_loss = has_loss != 0;
  st->ldr.clear();
  for (int64_t i = 0; i < n_hist; ++i) st->ldr.emplace_back(epochs[i], ldr[i]);
  return GTE_OK;
}

// thresholds and lag of a caller-held tuner state (the drop-in's TunerState)
int gte_tuner_load(gte_tuner* st, int64_t n_thresholds, const double* thresholds, int64_t delta) {
  if (n_thresholds < 1) return set_error(GTE_CONFIG, "tuner: empty threshold set");
  if (delta < 1) return set_error(GTE_CONFIG, "tuner: delta must be >= 1");
  st->thresholds.assign(thresholds, thresholds + n_thresholds);
  st->delta = delta;
  if (st->idx >= st->thresholds.size()) st->idx = st->thresholds.size() - 1;
  return GTE_OK;
}

int gte_tuner_destroy(gte_tuner* st) {
  delete st;
  return GTE_OK;
}

// select_k (reformation.cpp:267-275)
int gte_select_k(int64_t l2_bytes, int64_t hidden_dim, int64_t i, int64_t* out) {
  if (l2_bytes <= 0 || hidden_dim <= 0 || i <= 0) return set_error(GTE_CONFIG, "select_k: all arguments must be positive");
  const double raw = std::floor(std::sqrt((double)l2_bytes / ((double)i * (double)hidden_dim)));
  if (raw < 1.0) return set_error(GTE_CONFIG, "select_k: cache budget yields k < 1");
  *out = (int64_t)std::bit_floor((uint64_t)raw);
  return GTE_OK;
}

// select_db (reformation.cpp:277-296); entries ascending by d_b
int gte_select_db(int64_t n, const int64_t* db, const double* thr, int64_t* out) {
  if (n <= 0) return set_error(GTE_CONFIG, "select_db: empty profile");
  double best = -std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < n; ++i) best = std::max(best, thr[i]);
  const double median = (double)(n - 1) / 2.0;
  int64_t chosen = -1;
  double cd = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (thr[i] != best) continue;
    const double dist = std::abs((double)i - median);
    if (chosen == -1 || dist < cd || (dist == cd && db[i] > chosen)) {
      chosen = db[i];
      cd = dist;
    }
  }
  *out = chosen;
  return GTE_OK;
}

// check_conditions (interleave.cpp:68-99): C1 self-loops, C2 Dirac, C3
// double-sweep BFS bound. flags = {c1, c2_pass, c3}; ints = {layers,
// sweep_from, sweep_to, diameter_lower_bound}.
int gte_check_conditions(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t layers,
                         int32_t* flags, int64_t* ints) {
  (void)nnz;
  flags[0] = 1;
  for (int64_t u = 0; u < n && flags[0]; ++u)
    if (!std::binary_search(cols + row_off[u], cols + row_off[u + 1], u)) flags[0] = 0;
  std::vector<std::vector<int64_t>> adj((size_t)n);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = row_off[u]; e < row_off[u + 1]; ++e) {
      const int64_t v = cols[e];
      if (u == v) continue;
      adj[(size_t)u].push_back(v);
      adj[(size_t)v].push_back(u);
    }
  for (auto& nb : adj) {
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
  }
  int64_t min_deg = n == 0 ? 0 : (int64_t)adj[0].size();
  for (const auto& nb : adj) min_deg = std::min(min_deg, (int64_t)nb.size());
  flags[1] = (n >= 1 && 2 * min_deg >= n) ? 1 : 0;
  flags[2] = 0;
  ints[0] = layers;
  ints[1] = ints[2] = ints[3] = -1;
  if (n >= 1) {
    std::vector<int> dist((size_t)n);
    auto bfs = [&](int64_t src) {
      std::fill(dist.begin(), dist.end(), -1);
      std::vector<int64_t> fr{src}, nx;
      dist[(size_t)src] = 0;
      int64_t far = src;
      int far_d = 0;
      while (!fr.empty()) {
        nx.clear();
        for (int64_t u : fr)
          for (int64_t v : adj[(size_t)u])
            if (dist[(size_t)v] == -1) {
              dist[(size_t)v] = dist[(size_t)u] + 1;
              nx.push_back(v);
              if (dist[(size_t)v] > far_d || (dist[(size_t)v] == far_d && v < far)) {
                far_d = dist[(size_t)v];
                far = v;
              }
            }
        fr.swap(nx);
      }
      return far;
    };
    const int64_t u = bfs(0);
    const bool connected = std::find(dist.begin(), dist.end(), -1) == dist.end();
    const int64_t v = bfs(u);
    ints[1] = u;
    ints[2] = v;
    ints[3] = dist[(size_t)v];
    flags[2] = (connected && ints[3] <= layers) ? 1 : 0;
  }
  return GTE_OK;
}

// select_mode (interleave.cpp:101-106): mode 0 sparse / 1 dense; reason 0
// conditions_failed, 1 scheduled_dense, 2 conditions_passed
int gte_select_mode(const int32_t* flags, int64_t epoch, int64_t dense_period, int32_t* mode, int32_t* reason) {
  if (dense_period < 1) return set_error(GTE_CONFIG, "select_mode: dense_period must be >= 1");
  if (epoch % dense_period == 0) {
    *mode = 1;
    *reason = 1;
  } else if (!(flags[0] && flags[1] && flags[2])) {
    *mode = 1;
    *reason = 0;
  } else {
    *mode = 0;
    *reason = 2;
  }
  return GTE_OK;
}

// partition_sequence (parallel.cpp:96-113): ids[padded], worker w owns
// ids[w*per, (w+1)*per).
int gte_partition_sequence(int64_t seq_len, int64_t num_workers, uint64_t seed, int64_t* ids, int64_t* padded) {
  if (num_workers < 1) return set_error(GTE_CONFIG, "partition_sequence: worker count must be >= 1");
  if (seq_len < 1) return set_error(GTE_CONFIG, "partition_sequence: empty sequence");
  const int64_t pad = ((seq_len + num_workers - 1) / num_workers) * num_workers;
  std::vector<int64_t> v((size_t)pad);
  std::iota(v.begin(), v.end(), int64_t{0});
  std::mt19937_64 rng(seed);
  std::shuffle(v.begin(), v.end(), rng);
  if (ids) std::copy(v.begin(), v.end(), ids);
  if (padded) *padded = pad;
  return GTE_OK;
}

}  // extern "C"

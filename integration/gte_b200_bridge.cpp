// gte_b200_bridge.cpp — the reference-side binding of the B200 hot path.
//
// Compiled against the REFERENCE's own headers (/root/reference/proj/include,
// `gte::` API, unmodified), it defines every hot-path function of that API in
// terms of the C ABI in include/gte_b200.h. A maintainer drops this file into
// the reference build in place of attention.cpp / partition.cpp /
// reformation.cpp / parallel.cpp / interleave.cpp; here
// integration/Makefile links it with the reference's untouched out-of-scope
// objects (model, config, matrix, IO) whose hot-path duplicates are weakened,
// and with the reference's own unit tests, which then run on the GPU.
//
// Numbers are the reference's `Real = double`: attention runs the fp64
// conformance kernels (dtype GTE_F64). Errors come back as gte_status codes
// and are rethrown as the reference's exception types with its messages.
#include <algorithm>
#include <iterator>
#include <istream>
#include <ostream>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "gte/attention.hpp"
#include "gte/graph.hpp"
#include "gte/interleave.hpp"
#include "gte/parallel.hpp"
#include "gte/partition.hpp"
#include "gte/reformation.hpp"
#include "gte_b200.h"

namespace gte {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = gte_last_error();
  switch (rc) {
    case GTE_CONFIG: throw ConfigError(msg);
    case GTE_DATA: throw DataError(msg);
    case GTE_DIVERGENCE: throw DivergenceError(msg);
    default: throw std::runtime_error("gte_b200: " + msg);
  }
}

inline void ck(int rc) {
  if (rc != GTE_OK) rethrow(rc);
}

gte_ctx* ctx() {
  static std::once_flag once;
  static gte_ctx* c = nullptr;
  std::call_once(once, [] { ck(gte_ctx_create(0, &c)); });
  return c;
}

struct PlanHandle {
  gte_plan* p = nullptr;
  explicit PlanHandle(const AttnPattern& pat) {
    std::vector<Index> ro = pat.row_offsets;
    if (ro.empty()) ro.assign(static_cast<size_t>(pat.rows) + 1, 0);
    ck(gte_plan_create_host(ctx(), pat.rows, pat.nnz(), ro.data(), pat.cols.empty() ? nullptr : pat.cols.data(), &p));
  }
  ~PlanHandle() { gte_plan_destroy(p); }
  PlanHandle(const PlanHandle&) = delete;
  PlanHandle& operator=(const PlanHandle&) = delete;
};

// Device plans of the last few patterns, keyed by content (rows, nnz and a
// FNV-1a hash of offsets + columns): a Trainer calls the attention with the
// same layout every step, and a plan (int32 CSR + CSC + execution plan) is
// built once per layout instead of once per call.
std::shared_ptr<PlanHandle> plan_for(const AttnPattern& pat) {
  uint64_t h = 1469598103934665603ULL;
  auto mix = [&](const std::vector<Index>& v) {
    for (Index x : v) {
      h ^= static_cast<uint64_t>(x);
      h *= 1099511628211ULL;
    }
  };
  mix(pat.row_offsets);
  mix(pat.cols);
  struct Entry {
    uint64_t key;
    Index rows, nnz;
    std::shared_ptr<PlanHandle> plan;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;  // most recent last
  std::lock_guard<std::mutex> lock(mu);
  for (size_t i = 0; i < cache.size(); ++i)
    if (cache[i].key == h && cache[i].rows == pat.rows && cache[i].nnz == pat.nnz()) {
      Entry e = cache[i];
      cache.erase(cache.begin() + static_cast<std::ptrdiff_t>(i));
      cache.push_back(e);
      return e.plan;
    }
  auto plan = std::make_shared<PlanHandle>(pat);
  cache.push_back({h, pat.rows, pat.nnz(), plan});
  if (cache.size() > 8) cache.erase(cache.begin());
  return plan;
}

// device buffer through the library's C ABI (the bridge has no CUDA runtime)
struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) { ck(gte_dev_alloc(ctx(), static_cast<int64_t>(bytes), &p)); }
  DevMem(const void* host, size_t bytes) : DevMem(bytes) { ck(gte_copy_h2d(ctx(), p, host, static_cast<int64_t>(bytes))); }
  ~DevMem() { gte_dev_free(ctx(), p); }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
};

void check_shapes(const Matrix& q, const Matrix& k, const Matrix& v) {  // attention.cpp:12-18
  if (q.rows() != k.rows() || q.rows() != v.rows()) throw ConfigError("attention: Q/K/V row counts differ");
  if (q.cols() != k.cols()) throw ConfigError("attention: Q/K column counts differ");
  if (q.cols() < 1) throw ConfigError("attention: d_K must be >= 1");
}

// fwd over a plan, one or more heads; returns out + lse (host)
void run_fwd(const PlanHandle& plan, int H, Index dk, Index dv, const Real* q, const Real* k, const Real* v,
             const Real* bias, const Real* wm, Real* out, std::vector<Real>& lse, int flags) {
  lse.assign(static_cast<size_t>(plan.p ? 1 : 1) * 0, 0.0);
  int64_t rows = 0;
  gte_plan_shape(plan.p, &rows, nullptr, nullptr, nullptr);
  lse.assign(static_cast<size_t>(rows * H) + 1, 0.0);
  if (rows == 0) return;
  ck(gte_sparse_attn_fwd_host(ctx(), plan.p, GTE_F64, H, (int)dk, (int)dv, q, k, v, bias, wm, out, lse.data(), flags));
}

void run_bwd(const PlanHandle& plan, int H, Index dk, Index dv, const Real* q, const Real* k, const Real* v,
             const Real* out, const std::vector<Real>& lse, const Real* up, const Real* bias, const Real* wm,
             Real* dq, Real* dkk, Real* dvv, Real* dbias) {
  int64_t rows = 0;
  gte_plan_shape(plan.p, &rows, nullptr, nullptr, nullptr);
  if (rows == 0) return;
  ck(gte_sparse_attn_bwd_host(ctx(), plan.p, GTE_F64, H, (int)dk, (int)dv, q, k, v, out, lse.data(), up, bias, wm,
                              dq, dkk, dvv, dbias));
}

const Real* opt(std::span<const Real> s) { return s.empty() ? nullptr : s.data(); }

Graph with_payload(Graph out, const Graph& src) {
  out.features = src.features;
  out.labels = src.labels;
  out.graph_label = src.graph_label;
  return out;
}

}  // namespace

// ============================================================== graph.hpp

namespace {
std::string slurp(std::istream& in) { return std::string(std::istreambuf_iterator<char>(in), {}); }
}  // namespace

// graph.cpp:68-109: parsed in libgte_b200 (multi-threaded), CSR built on the GPU
Graph load_edge_list(std::istream& in, std::optional<Index> num_nodes_hint) {
  const std::string text = slurp(in);
  gte_edges* e = nullptr;
  ck(gte_parse_edge_list(text.data(), static_cast<int64_t>(text.size()), num_nodes_hint ? *num_nodes_hint : -1, &e));
  int64_t n = 0, m = 0;
  gte_edges_info(e, &n, &m);
  std::vector<std::pair<Index, Index>> edges(static_cast<size_t>(m));
  std::vector<int64_t> s(static_cast<size_t>(m)), d(static_cast<size_t>(m));
  gte_edges_copy(e, s.data(), d.data());
  gte_edges_destroy(e);
  for (int64_t i = 0; i < m; ++i) edges[static_cast<size_t>(i)] = {s[static_cast<size_t>(i)], d[static_cast<size_t>(i)]};
  return graph_from_edges(n, std::move(edges));
}

// graph.cpp:302-336 (GTF1)
Matrix load_features_binary(std::istream& in) {
  const std::string bytes = slurp(in);
  int64_t n = 0, f = 0;
  ck(gte_gtf1_decode(bytes.data(), static_cast<int64_t>(bytes.size()), &n, &f, nullptr));
  std::vector<float> buf(static_cast<size_t>(n * f) + 1);
  ck(gte_gtf1_decode(bytes.data(), static_cast<int64_t>(bytes.size()), &n, &f, buf.data()));
  Matrix m(n, f);
  for (int64_t i = 0; i < n * f; ++i) m.data()[i] = buf[static_cast<size_t>(i)];
  return m;
}

void save_features_binary(std::ostream& out, const Matrix& m) {
  std::vector<float> buf(static_cast<size_t>(m.rows() * m.cols()) + 1);
  for (Index i = 0; i < m.rows() * m.cols(); ++i) buf[static_cast<size_t>(i)] = static_cast<float>(m.data()[i]);
  int64_t len = 0;
  gte_gtf1_encode(m.rows(), m.cols(), buf.data(), nullptr, &len);
  std::string bytes(static_cast<size_t>(len), '\0');
  ck(gte_gtf1_encode(m.rows(), m.cols(), buf.data(), bytes.data(), &len));
  out.write(bytes.data(), static_cast<std::streamsize>(len));
}

// graph.cpp:49-66
Graph graph_from_edges(Index num_nodes, std::vector<std::pair<Index, Index>> edges) {
  std::vector<Index> s(edges.size()), d(edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    s[i] = edges[i].first;
    d[i] = edges[i].second;
  }
  Graph g;
  g.num_nodes = num_nodes;
  g.row_offsets.assign(static_cast<size_t>(std::max<Index>(num_nodes, 0)) + 1, 0);
  std::vector<Index> cols(edges.size() + 1);
  int64_t nnz = 0;
  ck(gte_graph_from_edges_host(ctx(), num_nodes, (int64_t)edges.size(), s.data(), d.data(), g.row_offsets.data(),
                               cols.data(), &nnz));
  cols.resize(static_cast<size_t>(nnz));
  g.col_indices = std::move(cols);
  return g;
}

// graph.cpp:127-149
Graph add_self_loops(const Graph& g) {
  Graph out;
  out.num_nodes = g.num_nodes;
  out.row_offsets.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  std::vector<Index> cols(static_cast<size_t>(g.nnz() + g.num_nodes) + 1);
  std::vector<Index> ro = g.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  int64_t nnz = 0;
  ck(gte_add_self_loops_host(ctx(), g.num_nodes, g.nnz(), ro.data(), g.col_indices.data(), out.row_offsets.data(),
                             cols.data(), &nnz));
  cols.resize(static_cast<size_t>(nnz));
  out.col_indices = std::move(cols);
  return with_payload(std::move(out), g);
}

// graph.cpp:151-155
Real density(const Graph& g) {
  if (g.num_nodes < 1) throw DataError("density: empty graph");
  return static_cast<Real>(g.nnz()) / (static_cast<Real>(g.num_nodes) * static_cast<Real>(g.num_nodes));
}

// ========================================================== attention.hpp

AttnPattern pattern_from_graph(const Graph& g) {  // attention.cpp:26-32
  AttnPattern p;
  p.rows = g.num_nodes;
  p.row_offsets = g.row_offsets;
  p.cols = g.col_indices;
  return p;
}

AttnPattern dense_pattern(Index n) {  // attention.cpp:34-44
  AttnPattern p;
  p.rows = n;
  p.row_offsets.resize(static_cast<size_t>(n) + 1);
  p.cols.resize(static_cast<size_t>(n * n));
  for (Index i = 0; i <= n; ++i) p.row_offsets[static_cast<size_t>(i)] = i * n;
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) p.cols[static_cast<size_t>(i * n + j)] = j;
  return p;
}

// attention.cpp:96-162
AttnResult sparse_attention(const Matrix& q, const Matrix& k, const Matrix& v, const AttnPattern& pat,
                            std::span<const Real> bias, std::span<const Real> weight_mult, bool forbid_empty_rows) {
  check_shapes(q, k, v);
  if (pat.rows != q.rows()) throw ConfigError("sparse_attention: pattern/sequence length mismatch");
  if (!bias.empty() && static_cast<Index>(bias.size()) != pat.nnz())
    throw ConfigError("sparse_attention: bias must cover exactly the attended pairs");
  if (!weight_mult.empty() && static_cast<Index>(weight_mult.size()) != pat.nnz())
    throw ConfigError("sparse_attention: weight_mult size mismatch");
  AttnResult res;
  res.output = Matrix(q.rows(), v.cols());
  auto plan = plan_for(pat);
  std::vector<Real> lse;
  run_fwd(*plan, 1, q.cols(), v.cols(), q.data(), k.data(), v.data(), opt(bias), opt(weight_mult), res.output.data(), lse,
          forbid_empty_rows ? GTE_FORBID_EMPTY_ROWS : 0);
  res.macs.score_macs = pat.nnz() * q.cols();
  res.macs.weight_macs = pat.nnz() * v.cols();
  return res;
}

// attention.cpp:164-172
AttnResult edge_sparse_attention(const Matrix& q, const Matrix& k, const Matrix& v, const Graph& g,
                                 std::span<const Real> bias, std::span<const Real> weight_mult) {
  if (g.num_nodes != q.rows()) throw ConfigError("edge_sparse_attention: graph/sequence length mismatch");
  return sparse_attention(q, k, v, pattern_from_graph(g), bias, weight_mult, true);
}

// attention.cpp:241-320
AttnGrads sparse_attention_backward(const Matrix& q, const Matrix& k, const Matrix& v, const AttnPattern& pat,
                                    std::span<const Real> bias, std::span<const Real> weight_mult,
                                    const Matrix& upstream) {
  check_shapes(q, k, v);
  const Index s = q.rows(), dk = q.cols(), dv = v.cols();
  if (pat.rows != s) throw ConfigError("sparse_attention_backward: pattern mismatch");
  if (upstream.rows() != s || upstream.cols() != dv)
    throw ConfigError("sparse_attention_backward: upstream shape mismatch");
  AttnGrads g;
  g.dq = Matrix(s, dk);
  g.dk = Matrix(s, dk);
  g.dv = Matrix(s, dv);
  g.dbias.assign(static_cast<size_t>(pat.nnz()), 0.0);
  const auto planp = plan_for(pat);
  const PlanHandle& plan = *planp;
  Matrix out(s, dv);
  std::vector<Real> lse;
  // softmax statistics from the same kernels (the reference recomputes them
  // inside its backward, attention.cpp:275-290); no finiteness check there
  run_fwd(plan, 1, dk, dv, q.data(), k.data(), v.data(), opt(bias), opt(weight_mult), out.data(), lse,
          GTE_IGNORE_NONFINITE);
  std::vector<Real> db(static_cast<size_t>(pat.nnz()) + 1, 0.0);
  run_bwd(plan, 1, dk, dv, q.data(), k.data(), v.data(), out.data(), lse, upstream.data(), opt(bias),
          opt(weight_mult), g.dq.data(), g.dk.data(), g.dv.data(), db.data());
  std::copy(db.begin(), db.begin() + pat.nnz(), g.dbias.begin());
  return g;
}

namespace {
void check_finite_matrix(const Matrix& m, const char* name) {  // attention.cpp:20-22
  if (!m.all_finite()) throw DataError(std::string("attention: non-finite ") + name);
}
}  // namespace

// attention.cpp:46-94 -> flash-style dense kernel (gte_dense_attn_fwd_host, f64)
AttnResult dense_attention(const Matrix& q, const Matrix& k, const Matrix& v, const Matrix* bias,
                           const Matrix* weight_mult) {
  check_shapes(q, k, v);
  check_finite_matrix(q, "Q");
  check_finite_matrix(k, "K");
  check_finite_matrix(v, "V");
  const Index s = q.rows();
  if (bias) {
    if (bias->rows() != s || bias->cols() != s) throw ConfigError("dense_attention: bias shape");
    check_finite_matrix(*bias, "bias");
  }
  if (weight_mult && (weight_mult->rows() != s || weight_mult->cols() != s))
    throw ConfigError("dense_attention: weight_mult shape");
  AttnResult res;
  res.output = Matrix(s, v.cols());
  ck(gte_dense_attn_fwd_host(ctx(), GTE_F64, s, s, 1, static_cast<int>(q.cols()), static_cast<int>(v.cols()),
                                  q.data(), k.data(), v.data(), bias ? bias->data() : nullptr,
                                  weight_mult ? weight_mult->data() : nullptr, res.output.data(), nullptr));
  res.macs.score_macs = s * s * q.cols();
  res.macs.weight_macs = s * s * v.cols();
  return res;
}

// attention.cpp:174-239 -> flash-style dense backward (gte_dense_attn_bwd_host, f64)
AttnGrads dense_attention_backward(const Matrix& q, const Matrix& k, const Matrix& v, const Matrix* bias,
                                   const Matrix* weight_mult, const Matrix& upstream) {
  check_shapes(q, k, v);
  const Index s = q.rows(), dk = q.cols(), dv = v.cols();
  if (upstream.rows() != s || upstream.cols() != dv)
    throw ConfigError("dense_attention_backward: upstream shape mismatch");
  AttnGrads g;
  g.dq = Matrix(s, dk);
  g.dk = Matrix(s, dk);
  g.dv = Matrix(s, dv);
  g.dbias.assign(static_cast<size_t>(s * s), 0.0);
  if (s == 0) return g;
  ck(gte_dense_attn_bwd_host(ctx(), GTE_F64, s, s, 1, static_cast<int>(dk), static_cast<int>(dv), q.data(),
                                  k.data(), v.data(), bias ? bias->data() : nullptr,
                                  weight_mult ? weight_mult->data() : nullptr, upstream.data(), g.dq.data(),
                                  g.dk.data(), g.dv.data(), g.dbias.data()));
  return g;
}

// ========================================================== partition.hpp

Permutation Permutation::identity(Index n) {  // partition.cpp:395-402
  Permutation p;
  p.forward.resize(static_cast<size_t>(n));
  p.inverse.resize(static_cast<size_t>(n));
  std::iota(p.forward.begin(), p.forward.end(), Index{0});
  std::iota(p.inverse.begin(), p.inverse.end(), Index{0});
  return p;
}

bool Permutation::valid() const {  // partition.cpp:404-411
  if (forward.size() != inverse.size()) return false;
  for (Index i = 0; i < size(); ++i) {
    const Index f = forward[static_cast<size_t>(i)];
    if (f < 0 || f >= size() || inverse[static_cast<size_t>(f)] != i) return false;
  }
  return true;
}

// partition.cpp:458-493
void save_permutation(std::ostream& out, const Permutation& p) {
  std::string text;
  for (Index old = 0; old < p.size(); ++old)
    text += std::to_string(old) + " " + std::to_string(p.forward[static_cast<size_t>(old)]) + "\n";
  out << text;
}

Permutation load_permutation(std::istream& in) {
  const std::string text = slurp(in);
  int64_t n = 0;
  ck(gte_parse_permutation(text.data(), static_cast<int64_t>(text.size()), &n, nullptr, nullptr));
  Permutation p;
  p.forward.assign(static_cast<size_t>(n), -1);
  p.inverse.assign(static_cast<size_t>(n), -1);
  ck(gte_parse_permutation(text.data(), static_cast<int64_t>(text.size()), &n, p.forward.data(), p.inverse.data()));
  return p;
}

// partition.cpp:413-433 (device coarsening + host greedy passes in libgte_b200)
Permutation reorder(const Graph& g, Index k, std::uint64_t seed) {
  Permutation p;
  p.forward.resize(static_cast<size_t>(g.num_nodes));
  p.inverse.resize(static_cast<size_t>(g.num_nodes));
  std::vector<Index> ro = g.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  ck(gte_reorder(g.num_nodes, g.nnz(), ro.data(), g.col_indices.data(), k, seed, p.forward.data(),
                 p.inverse.data()));
  return p;
}

// partition.cpp:435-456
Graph permute_graph(const Graph& g, const Permutation& p) {
  if (p.size() != g.num_nodes || !p.valid()) throw ConfigError("permute_graph: bad permutation");
  Graph out;
  out.num_nodes = g.num_nodes;
  out.row_offsets.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  out.col_indices.assign(static_cast<size_t>(g.nnz()), 0);
  std::vector<Index> ro = g.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  ck(gte_permute_graph_host(ctx(), g.num_nodes, g.nnz(), ro.data(), g.col_indices.data(), p.forward.data(),
                            out.row_offsets.data(), out.col_indices.data()));
  if (!g.features.empty()) {
    out.features = Matrix(g.num_nodes, g.features.cols());
    for (Index u = 0; u < g.num_nodes; ++u) {
      auto src = g.features.row(u);
      std::copy(src.begin(), src.end(), out.features.row(p.forward[static_cast<size_t>(u)]).begin());
    }
  }
  if (!g.labels.empty()) {
    out.labels.resize(static_cast<size_t>(g.num_nodes));
    for (Index u = 0; u < g.num_nodes; ++u)
      out.labels[static_cast<size_t>(p.forward[static_cast<size_t>(u)])] = g.labels[static_cast<size_t>(u)];
  }
  out.graph_label = g.graph_label;
  return out;
}

std::vector<Index> cluster_boundaries(Index n, Index k) {  // partition.cpp:495-500
  std::vector<Index> b(static_cast<size_t>(k) + 1, 0);
  ck(gte_cluster_boundaries(n, k, b.data()));
  return b;
}

Index ClusterGrid::cluster_of(Index pos) const {  // partition.cpp:502-508
  const Index n = boundaries.back();
  const Index base = n / k, rem = n % k, cut = rem * (base + 1);
  if (pos < cut) return pos / (base + 1);
  return rem + (pos - cut) / base;
}

std::int64_t ClusterGrid::total_nnz() const {
  return std::accumulate(cell_nnz.begin(), cell_nnz.end(), std::int64_t{0});
}

// partition.cpp:514-539
ClusterGrid build_cluster_grid(const Graph& g, const Permutation& p, Index k) {
  if (k < 1 || k > g.num_nodes) throw ConfigError("build_cluster_grid: invalid k");
  if (p.size() != g.num_nodes || !p.valid()) throw ConfigError("build_cluster_grid: permutation does not match graph");
  ClusterGrid grid;
  grid.k = k;
  grid.boundaries.assign(static_cast<size_t>(k) + 1, 0);
  grid.cell_nnz.assign(static_cast<size_t>(k * k), 0);
  grid.cell_density.assign(static_cast<size_t>(k * k), 0.0);
  std::vector<Index> ro = g.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(g.num_nodes) + 1, 0);
  ck(gte_build_cluster_grid_host(ctx(), g.num_nodes, g.nnz(), ro.data(), g.col_indices.data(), p.forward.data(), k,
                                 grid.boundaries.data(), grid.cell_nnz.data(), grid.cell_density.data()));
  return grid;
}

Real diagonal_edge_fraction(const ClusterGrid& grid) {  // partition.cpp:541-547
  Real out = 0;
  ck(gte_diagonal_edge_fraction(grid.k, grid.cell_nnz.data(), &out));
  return out;
}

// ======================================================== reformation.hpp

Index ClusterSparseLayout::transferred_cells() const {
  return static_cast<Index>(std::count(cell_state.begin(), cell_state.end(), CellState::Transferred));
}

std::int64_t ClusterSparseLayout::subblock_count() const {
  std::int64_t n = 0;
  for (const auto& b : cell_blocks) n += static_cast<std::int64_t>(b.size());
  return n;
}

// reformation.cpp:56-109 (exact lazy-heap packer in libgte_b200)
std::vector<SubBlock> pack_subblocks(std::span<const std::pair<Index, Index>> cell_edges, Index n_rows, Index n_cols,
                                     Index d_b) {
  std::vector<Index> r(cell_edges.size() + 1), c(cell_edges.size() + 1);
  for (size_t i = 0; i < cell_edges.size(); ++i) {
    r[i] = cell_edges[i].first;
    c[i] = cell_edges[i].second;
  }
  const Index cap = d_b >= 1 ? (static_cast<Index>(cell_edges.size()) + d_b * d_b - 1) / (d_b * d_b) : 0;
  std::vector<Index> t(static_cast<size_t>(2 * cap) + 2);
  int64_t nt = 0;
  ck(gte_pack_subblocks(static_cast<int64_t>(cell_edges.size()), r.data(), c.data(), n_rows, n_cols, d_b, t.data(), &nt));
  std::vector<SubBlock> tiles(static_cast<size_t>(nt));
  for (int64_t i = 0; i < nt; ++i) tiles[static_cast<size_t>(i)] = SubBlock{t[2 * i], t[2 * i + 1]};
  return tiles;
}

// reformation.cpp:111-195
ClusterSparseLayout build_layout(const ClusterGrid& grid, const Graph& g_perm, TransferStrategy strategy,
                                 Real beta_thre, Real beta_g, Index d_b) {
  const Index k = grid.k, n = g_perm.num_nodes;
  if (grid.boundaries.back() != n) throw ConfigError("build_layout: grid/graph size mismatch");
  if (grid.total_nnz() != g_perm.nnz()) throw ConfigError("build_layout: grid/graph nnz mismatch");
  std::vector<Index> ro = g_perm.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(n) + 1, 0);
  gte_layout* L = nullptr;
  ck(gte_build_layout_host(ctx(), n, g_perm.nnz(), ro.data(), g_perm.col_indices.data(), k, grid.boundaries.data(),
                           grid.cell_nnz.data(), grid.cell_density.data(),
                           strategy == TransferStrategy::Indolent ? 0 : 1, beta_thre, beta_g, d_b, &L));
  std::unique_ptr<gte_layout, int (*)(gte_layout*)> hold(L, gte_layout_destroy);
  int64_t transferred = 0, nb = 0, dropped = 0, pnnz = 0;
  gte_layout_info(L, &transferred, &nb, &dropped, &pnnz);
  std::vector<int32_t> state(static_cast<size_t>(k * k));
  std::vector<int64_t> boff(static_cast<size_t>(k * k) + 1), blocks(static_cast<size_t>(2 * nb) + 2);
  gte_layout_cells(L, state.data(), boff.data(), blocks.data());
  ClusterSparseLayout out;
  out.seq_len = n;
  out.k = k;
  out.d_b = d_b;
  out.boundaries = grid.boundaries;
  out.cell_state.resize(static_cast<size_t>(k * k));
  out.cell_blocks.resize(static_cast<size_t>(k * k));
  for (Index cell = 0; cell < k * k; ++cell) {
    out.cell_state[static_cast<size_t>(cell)] = state[static_cast<size_t>(cell)] ? CellState::Transferred : CellState::Untouched;
    for (int64_t b = boff[static_cast<size_t>(cell)]; b < boff[static_cast<size_t>(cell) + 1]; ++b)
      out.cell_blocks[static_cast<size_t>(cell)].push_back(SubBlock{blocks[2 * b], blocks[2 * b + 1]});
  }
  out.dropped_edges = dropped;
  out.pattern.rows = n;
  out.pattern.row_offsets.assign(static_cast<size_t>(n) + 1, 0);
  out.pattern.cols.assign(static_cast<size_t>(pnnz), 0);
  std::vector<Index> tmp(static_cast<size_t>(pnnz) + 1);
  ck(gte_layout_pattern_host(L, out.pattern.row_offsets.data(), tmp.data()));
  std::copy(tmp.begin(), tmp.begin() + pnnz, out.pattern.cols.begin());
  return out;
}

// reformation.cpp:197-204
AttnResult cluster_sparse_attention(const Matrix& q, const Matrix& k, const Matrix& v, const ClusterSparseLayout& layout,
                                    std::span<const Real> bias, std::span<const Real> weight_mult) {
  if (layout.seq_len != q.rows()) throw ConfigError("cluster_sparse_attention: layout/sequence length mismatch");
  return sparse_attention(q, k, v, layout.pattern, bias, weight_mult);
}

// reformation.cpp:224-265
TunerState make_tuner_state(Real beta_g, Index delta) {
  gte_tuner* t = nullptr;
  ck(gte_tuner_create(beta_g, delta, &t));
  TunerState st;
  double thr[8];
  int64_t n = 0, idx = 0;
  int32_t has = 0;
  gte_tuner_state(t, &st.avg_loss, &idx, thr, &n, &has);
  gte_tuner_destroy(t);
  st.thresholds.assign(thr, thr + n);
  st.idx = static_cast<size_t>(idx);
  st.delta = delta;
  st.has_loss = has != 0;
  return st;
}

// reformation.cpp:240-265: the caller-owned TunerState goes through the
// library's controller (gte_tuner_update) and comes back updated.
void tuner_update(TunerState& state, Real loss, Real epoch_time_s, Index epoch) {
  gte_tuner* t = nullptr;
  ck(gte_tuner_create(0.5, 1, &t));
  std::unique_ptr<gte_tuner, int (*)(gte_tuner*)> hold(t, gte_tuner_destroy);
  std::vector<int64_t> ep;
  std::vector<double> ldr;
  for (const auto& [e, v] : state.ldr_history) {
    ep.push_back(e);
    ldr.push_back(v);
  }
  ck(gte_tuner_set(t, state.avg_loss, static_cast<int64_t>(state.idx), state.has_loss ? 1 : 0,
                   static_cast<int64_t>(ep.size()), ep.data(), ldr.data()));
  ck(gte_tuner_load(t, static_cast<int64_t>(state.thresholds.size()), state.thresholds.data(), state.delta));
  ck(gte_tuner_update(t, loss, epoch_time_s, epoch));
  std::vector<double> thr(state.thresholds.size() + 1);
  int64_t n_thr = 0, idx = 0, n_hist = 0;
  int32_t has = 0;
  gte_tuner_state(t, &state.avg_loss, &idx, thr.data(), &n_thr, &has);
  state.idx = static_cast<size_t>(idx);
  state.has_loss = has != 0;
  gte_tuner_history(t, nullptr, nullptr, &n_hist);
  ep.assign(static_cast<size_t>(n_hist), 0);
  ldr.assign(static_cast<size_t>(n_hist), 0.0);
  gte_tuner_history(t, ep.data(), ldr.data(), &n_hist);
  state.ldr_history.clear();
  for (int64_t i = 0; i < n_hist; ++i) state.ldr_history.emplace_back(ep[static_cast<size_t>(i)], ldr[static_cast<size_t>(i)]);
}

Index select_k(std::int64_t l2_bytes, Index hidden_dim, Index i) {
  int64_t out = 0;
  ck(gte_select_k(l2_bytes, hidden_dim, i, &out));
  return out;
}

Index select_db(const std::map<Index, Real>& profile) {
  std::vector<int64_t> db;
  std::vector<double> thr;
  for (const auto& [d, t] : profile) {
    db.push_back(d);
    thr.push_back(t);
  }
  int64_t out = 0;
  ck(gte_select_db(static_cast<int64_t>(db.size()), db.data(), thr.data(), &out));
  return out;
}

// ========================================================= interleave.hpp

const char* to_string(Mode m) { return m == Mode::Sparse ? "sparse" : "dense"; }

const char* to_string(ModeReason r) {
  switch (r) {
    case ModeReason::ConditionsFailed: return "conditions_failed";
    case ModeReason::ScheduledDense: return "scheduled_dense";
    case ModeReason::ConditionsPassed: return "conditions_passed";
  }
  return "?";
}

ConditionReport check_conditions(const Graph& g_seq, Index layers) {  // interleave.cpp:68-99
  int32_t flags[3] = {0, 0, 0};
  int64_t ints[4] = {0, -1, -1, -1};
  std::vector<Index> ro = g_seq.row_offsets;
  if (ro.empty()) ro.assign(static_cast<size_t>(g_seq.num_nodes) + 1, 0);
  ck(gte_check_conditions(g_seq.num_nodes, g_seq.nnz(), ro.data(), g_seq.col_indices.data(), layers, flags, ints));
  ConditionReport rep;
  rep.c1_self_attend = flags[0] != 0;
  rep.c2_hamiltonian = flags[1] ? HamiltonianCheck::Pass : HamiltonianCheck::Unknown;
  rep.c3_reachable_within_l = flags[2] != 0;
  rep.layers = ints[0];
  rep.sweep_from = ints[1];
  rep.sweep_to = ints[2];
  rep.diameter_lower_bound = ints[3];
  return rep;
}

AttentionMode select_mode(const ConditionReport& report, Index epoch, Index dense_period) {  // interleave.cpp:101-106
  const int32_t flags[3] = {report.c1_self_attend ? 1 : 0, report.c2_hamiltonian == HamiltonianCheck::Pass ? 1 : 0,
                            report.c3_reachable_within_l ? 1 : 0};
  int32_t mode = 1, reason = 0;
  ck(gte_select_mode(flags, epoch, dense_period, &mode, &reason));
  return {mode == 0 ? Mode::Sparse : Mode::Dense,
          reason == 1 ? ModeReason::ScheduledDense : (reason == 2 ? ModeReason::ConditionsPassed : ModeReason::ConditionsFailed)};
}

// =========================================================== parallel.hpp

void CommLedger::accumulate(const CommLedger& other) {  // parallel.cpp:83-94
  if (workers.size() != other.workers.size()) throw ConfigError("ledger: worker count mismatch");
  for (size_t w = 0; w < workers.size(); ++w) {
    workers[w].qkv_gather += other.workers[w].qkv_gather;
    workers[w].qkv_gather_cross += other.workers[w].qkv_gather_cross;
    workers[w].output_scatter += other.workers[w].output_scatter;
    workers[w].output_scatter_cross += other.workers[w].output_scatter_cross;
    workers[w].bias_exchange += other.workers[w].bias_exchange;
  }
}

std::vector<WorkerShard> partition_sequence(Index seq_len, Index num_workers, std::uint64_t seed) {  // parallel.cpp:96-113
  int64_t padded = 0;
  if (num_workers >= 1 && seq_len >= 1) padded = ((seq_len + num_workers - 1) / num_workers) * num_workers;
  std::vector<Index> ids(static_cast<size_t>(padded) + 1);
  ck(gte_partition_sequence(seq_len, num_workers, seed, ids.data(), &padded));
  const Index per = padded / num_workers;
  std::vector<WorkerShard> shards(static_cast<size_t>(num_workers));
  for (Index w = 0; w < num_workers; ++w) {
    shards[static_cast<size_t>(w)].worker_id = w;
    shards[static_cast<size_t>(w)].token_ids.assign(ids.begin() + w * per, ids.begin() + (w + 1) * per);
  }
  return shards;
}

namespace {

struct ShardShape {
  Index num_workers = 0, rows = 0, d = 0, total = 0;
};

ShardShape validate_shards(const std::vector<Matrix>& mats, std::span<const std::vector<Index>> token_ids) {  // parallel.cpp:18-37
  if (mats.empty() || mats.size() != token_ids.size()) throw ConfigError("all_to_all: shard count mismatch");
  ShardShape s;
  s.num_workers = static_cast<Index>(mats.size());
  s.rows = mats[0].rows();
  s.d = mats[0].cols();
  for (size_t w = 0; w < mats.size(); ++w) {
    if (mats[w].rows() != s.rows || mats[w].cols() != s.d) throw ConfigError("all_to_all: ragged shards");
    if (static_cast<Index>(token_ids[w].size()) != s.rows) throw ConfigError("all_to_all: token ids misaligned with shard rows");
  }
  s.total = s.rows * s.num_workers;
  return s;
}

void check_divisibility(Index d, Index num_heads, Index num_workers) {  // parallel.cpp:39-46
  if (num_heads % num_workers != 0) throw ConfigError("all_to_all: head count not divisible by worker count");
  if (d % num_heads != 0) throw ConfigError("all_to_all: hidden dim not divisible by head count");
}

void ledger_add(CommLedger* ledger, Index src, Index dst, std::int64_t elems, bool as_qkv) {
  if (!ledger) return;
  auto& e = ledger->workers[static_cast<size_t>(src)];
  if (as_qkv) {
    e.qkv_gather += elems;
    if (dst != src) e.qkv_gather_cross += elems;
  } else {
    e.output_scatter += elems;
    if (dst != src) e.output_scatter_cross += elems;
  }
}

}  // namespace

// parallel.cpp:115-147 (in-process exchange + element ledger)
std::vector<Matrix> all_to_all_seq_to_head(const std::vector<Matrix>& shard_mats,
                                           std::span<const std::vector<Index>> token_ids, Index num_heads,
                                           CommLedger* ledger, bool count_as_qkv) {
  ShardShape s = validate_shards(shard_mats, token_ids);
  check_divisibility(s.d, num_heads, s.num_workers);
  const Index slice = s.d / s.num_workers;
  std::vector<Matrix> out(static_cast<size_t>(s.num_workers), Matrix(s.total, slice));
  for (Index src = 0; src < s.num_workers; ++src) {
    const Matrix& m = shard_mats[static_cast<size_t>(src)];
    for (Index dst = 0; dst < s.num_workers; ++dst) {
      Matrix& o = out[static_cast<size_t>(dst)];
      for (Index r = 0; r < s.rows; ++r) {
        const Index token = token_ids[static_cast<size_t>(src)][static_cast<size_t>(r)];
        std::copy(m.data() + r * s.d + dst * slice, m.data() + r * s.d + (dst + 1) * slice, o.data() + token * slice);
      }
      ledger_add(ledger, src, dst, static_cast<std::int64_t>(s.rows) * slice, count_as_qkv);
    }
  }
  return out;
}

// parallel.cpp:149-188
std::vector<Matrix> all_to_all_head_to_seq(const std::vector<Matrix>& head_slices,
                                           std::span<const std::vector<Index>> token_ids, CommLedger* ledger,
                                           bool count_as_scatter) {
  if (head_slices.empty() || head_slices.size() != token_ids.size()) throw ConfigError("all_to_all: shard count mismatch");
  const Index nw = static_cast<Index>(head_slices.size());
  const Index total = head_slices[0].rows(), slice = head_slices[0].cols();
  for (const Matrix& m : head_slices)
    if (m.rows() != total || m.cols() != slice) throw ConfigError("all_to_all: ragged slices");
  const Index rows = total / nw;
  if (rows * nw != total) throw ConfigError("all_to_all: sequence not divisible");
  std::vector<Matrix> out(static_cast<size_t>(nw), Matrix(rows, slice * nw));
  for (Index src = 0; src < nw; ++src) {
    const Matrix& m = head_slices[static_cast<size_t>(src)];
    for (Index dst = 0; dst < nw; ++dst) {
      Matrix& o = out[static_cast<size_t>(dst)];
      for (Index r = 0; r < rows; ++r) {
        const Index token = token_ids[static_cast<size_t>(dst)][static_cast<size_t>(r)];
        std::copy(m.data() + token * slice, m.data() + (token + 1) * slice, o.data() + r * o.cols() + src * slice);
      }
      ledger_add(ledger, src, dst, static_cast<std::int64_t>(rows) * slice, !count_as_scatter);
    }
  }
  return out;
}

namespace {

// P in-process workers of the distributed layer on the device (gte_sp_layer
// with the loopback exchange): shards uploaded once, the Ulysses all-to-alls,
// the cluster permutation and the per-worker H/P heads all in libgte_b200.
struct DeviceLayer {
  Index P, rows, d;
  std::shared_ptr<PlanHandle> plan;
  gte_sp* sp = nullptr;
  gte_sp_layer* L = nullptr;
  std::vector<std::unique_ptr<DevMem>> in, out, dq, dk, dv;
  std::unique_ptr<DevMem> bias_d, wm_d;

  DeviceLayer(const std::vector<std::vector<Index>>& ids, const Permutation& perm, const AttnPattern& pattern,
              Index num_heads, Index d_)
      : P(static_cast<Index>(ids.size())), rows(static_cast<Index>(ids[0].size())), d(d_) {
    plan = plan_for(pattern);
    std::vector<int64_t> tok;
    for (const auto& t : ids) tok.insert(tok.end(), t.begin(), t.end());
    ck(gte_sp_create(ctx(), P, rows, tok.data(), perm.forward.data(), &sp));
    ck(gte_sp_layer_create(ctx(), sp, plan->p, nullptr, 0, GTE_F64, num_heads, d, &L));
  }
  ~DeviceLayer() {
    gte_sp_layer_destroy(L);
    gte_sp_destroy(sp);
  }
  std::vector<void*> upload(const std::vector<Matrix>& mats) {
    std::vector<void*> ptrs;
    for (const Matrix& m : mats) {
      in.push_back(std::make_unique<DevMem>(m.data(), sizeof(Real) * static_cast<size_t>(rows * d)));
      ptrs.push_back(in.back()->p);
    }
    return ptrs;
  }
  std::vector<void*> make(std::vector<std::unique_ptr<DevMem>>& into) {
    std::vector<void*> ptrs;
    for (Index w = 0; w < P; ++w) {
      into.push_back(std::make_unique<DevMem>(sizeof(Real) * static_cast<size_t>(rows * d)));
      ptrs.push_back(into.back()->p);
    }
    return ptrs;
  }
  void put_bias(std::span<const Real> bias, std::span<const Real> wm) {
    if (!bias.empty() && !bias_d) bias_d = std::make_unique<DevMem>(bias.data(), sizeof(Real) * bias.size());
    if (!wm.empty() && !wm_d) wm_d = std::make_unique<DevMem>(wm.data(), sizeof(Real) * wm.size());
  }
  void forward(const std::vector<Matrix>& q, const std::vector<Matrix>& k, const std::vector<Matrix>& v,
               std::span<const Real> bias, std::span<const Real> wm, int flags) {
    put_bias(bias, wm);
    const auto qp = upload(q), kp = upload(k), vp = upload(v);
    const auto op = make(out);
    ck(gte_sp_layer_fwd(L, qp.data(), kp.data(), vp.data(), bias_d ? bias_d->p : nullptr, wm_d ? wm_d->p : nullptr,
                        op.data(), flags));
    ck(gte_ctx_sync(ctx()));  // data-dependent errors (attention.cpp:20-22, 119-123)
  }
  void backward(const std::vector<Matrix>& up, std::span<const Real> bias, std::span<const Real> wm, Real* dbias) {
    put_bias(bias, wm);
    const auto upp = upload(up);
    const auto a = make(dq), b = make(dk), c = make(dv);
    DevMem db(sizeof(Real) * static_cast<size_t>(plan_nnz() + 1));
    ck(gte_sp_layer_bwd(L, upp.data(), bias_d ? bias_d->p : nullptr, wm_d ? wm_d->p : nullptr, a.data(), b.data(),
                        c.data(), db.p));
    ck(gte_copy_d2h(ctx(), dbias, db.p, static_cast<int64_t>(sizeof(Real) * plan_nnz())));
  }
  int64_t plan_nnz() const {
    int64_t nnz = 0;
    gte_plan_shape(plan->p, nullptr, &nnz, nullptr, nullptr);
    return nnz;
  }
  std::vector<Matrix> download(const std::vector<std::unique_ptr<DevMem>>& bufs, Index cols) {
    std::vector<Matrix> res;
    for (const auto& b : bufs) {
      Matrix m(rows, cols);
      ck(gte_copy_d2h(ctx(), m.data(), b->p, static_cast<int64_t>(sizeof(Real) * static_cast<size_t>(rows * cols))));
      res.push_back(std::move(m));
    }
    return res;
  }
};

}  // namespace

// parallel.cpp:190-252: exchange accounting as the reference; the workers'
// exchanges and heads run on the device (gte_sp_layer, loopback exchange).
DistAttnResult run_distributed_layer(const std::vector<WorkerShard>& shards, const AttnPattern& pattern,
                                     const Permutation& perm, Index num_heads, std::span<const Real> bias,
                                     std::span<const Real> weight_mult, CommLedger& ledger) {
  if (shards.empty()) throw ConfigError("run_distributed_layer: no shards");
  const Index nw = static_cast<Index>(shards.size());
  if (static_cast<Index>(ledger.workers.size()) != nw)
    throw ConfigError("run_distributed_layer: ledger sized for wrong worker count");
  std::vector<Matrix> qm, km, vm;
  std::vector<std::vector<Index>> ids;
  for (const WorkerShard& sh : shards) {
    qm.push_back(sh.q_sub);
    km.push_back(sh.k_sub);
    vm.push_back(sh.v_sub);
    ids.push_back(sh.token_ids);
  }
  const Index d = qm[0].cols();
  const Index total = qm[0].rows() * nw;
  if (pattern.rows != total) throw ConfigError("run_distributed_layer: pattern/sequence mismatch");
  if (perm.size() != total) throw ConfigError("run_distributed_layer: permutation size mismatch");
  check_divisibility(d, num_heads, nw);
  const Index hd = d / num_heads;
  if (!weight_mult.empty() && static_cast<Index>(weight_mult.size()) != num_heads * pattern.nnz())
    throw ConfigError("run_distributed_layer: weight_mult size mismatch");
  // seq -> head exchanges of Q, K, V (validation + ledger, parallel.cpp:219-221)
  for (const auto* mats : {&qm, &km, &vm}) {
    ShardShape s = validate_shards(*mats, ids);
    for (Index src = 0; src < nw; ++src)
      for (Index dst = 0; dst < nw; ++dst) ledger_add(&ledger, src, dst, static_cast<std::int64_t>(s.rows) * (d / nw), true);
  }
  if (!bias.empty())
    for (auto& e : ledger.workers) e.bias_exchange += static_cast<std::int64_t>(bias.size());
  // the layer on the device: Ulysses exchange + per-worker heads (gte_sp_layer)
  DeviceLayer layer(ids, perm, pattern, num_heads, d);
  layer.forward(qm, km, vm, bias, weight_mult, 0);
  DistAttnResult res;
  res.macs.score_macs = pattern.nnz() * hd * num_heads;
  res.macs.weight_macs = pattern.nnz() * hd * num_heads;
  res.out_shards = layer.download(layer.out, d);
  // head -> seq exchange of O (parallel.cpp:250)
  for (Index src = 0; src < nw; ++src)
    for (Index dst = 0; dst < nw; ++dst) ledger_add(&ledger, src, dst, static_cast<std::int64_t>(total / nw) * (d / nw), false);
  return res;
}

// parallel.cpp:254-269
DistAttnResult run_distributed_layer(const std::vector<WorkerShard>& shards, const Graph* g_exec, AttentionMode mode,
                                     const ClusterSparseLayout* layout, const Permutation& perm, Index num_heads,
                                     CommLedger& ledger) {
  AttnPattern pattern;
  if (mode.mode == Mode::Dense) {
    pattern = dense_pattern(perm.size());
  } else if (layout != nullptr) {
    pattern = layout->pattern;
  } else if (g_exec != nullptr) {
    pattern = pattern_from_graph(*g_exec);
  } else {
    throw ConfigError("run_distributed_layer: sparse mode without a graph");
  }
  return run_distributed_layer(shards, pattern, perm, num_heads, {}, {}, ledger);
}

// parallel.cpp:271-332
DistAttnGrads run_distributed_layer_backward(const std::vector<WorkerShard>& shards, const AttnPattern& pattern,
                                             const Permutation& perm, Index num_heads, std::span<const Real> bias,
                                             std::span<const Real> weight_mult,
                                             const std::vector<Matrix>& upstream_shards) {
  const Index nw = static_cast<Index>(shards.size());
  std::vector<Matrix> qm, km, vm;
  std::vector<std::vector<Index>> ids;
  for (const WorkerShard& sh : shards) {
    qm.push_back(sh.q_sub);
    km.push_back(sh.k_sub);
    vm.push_back(sh.v_sub);
    ids.push_back(sh.token_ids);
  }
  const Index d = qm[0].cols();
  const Index total = qm[0].rows() * nw;
  check_divisibility(d, num_heads, nw);
  const Index hd = d / num_heads;
  for (const std::vector<Matrix>* mats : std::initializer_list<const std::vector<Matrix>*>{&qm, &km, &vm, &upstream_shards}) validate_shards(*mats, ids);
  if (pattern.rows != total) throw ConfigError("run_distributed_layer: pattern/sequence mismatch");
  if (perm.size() != total) throw ConfigError("run_distributed_layer: permutation size mismatch");
  (void)hd;
  DeviceLayer layer(ids, perm, pattern, num_heads, d);
  layer.forward(qm, km, vm, bias, weight_mult, GTE_IGNORE_NONFINITE);  // no finiteness check in the backward
  std::vector<Real> db(static_cast<size_t>(pattern.nnz()) + 1, 0.0);
  layer.backward(upstream_shards, bias, weight_mult, db.data());
  DistAttnGrads g;
  g.dbias.assign(db.begin(), db.begin() + pattern.nnz());
  g.dq_sub = layer.download(layer.dq, d);
  g.dk_sub = layer.download(layer.dk, d);
  g.dv_sub = layer.download(layer.dv, d);
  return g;
}

}  // namespace gte

// TEST INFRASTRUCTURE — not product code.
//
// A C ABI over the *compiled reference* (oracle/_ref/libgte_ref.a, built from
// /root/reference/proj/src by oracle/Makefile) so that Python can generate
// golden fixtures and pin the C restatement against the real thing. Only
// tests/golden/make_golden.py and tests/ load it. Nothing here re-implements
// the algorithm: every entry forwards to the reference gte:: function named in
// its comment.
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "gte/attention.hpp"
#include "gte/graph.hpp"
#include "gte/interleave.hpp"
#include "gte/model.hpp"
#include "gte/parallel.hpp"
#include "gte/partition.hpp"
#include "gte/reformation.hpp"
#include "oracles.hpp"  // reference test oracles (random_graph)

using namespace gte;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

struct CCsr {
  int64_t n, nnz;
  int64_t* row_off;
  int64_t* cols;
};

int64_t* dup_vec(const std::vector<Index>& v) {
  auto* p = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (v.size() + 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(int64_t) * v.size());
  return p;
}

void to_c(const Graph& g, CCsr* out) {
  out->n = g.num_nodes;
  out->nnz = g.nnz();
  out->row_off = dup_vec(g.row_offsets);
  out->cols = dup_vec(g.col_indices);
}

void to_c(const AttnPattern& p, CCsr* out) {
  out->n = p.rows;
  out->nnz = p.nnz();
  out->row_off = dup_vec(p.row_offsets);
  out->cols = dup_vec(p.cols);
}

Graph from_c(const CCsr* c) {
  Graph g;
  g.num_nodes = c->n;
  g.row_offsets.assign(c->row_off, c->row_off + c->n + 1);
  g.col_indices.assign(c->cols, c->cols + c->nnz);
  return g;
}

AttnPattern pat_from_c(const CCsr* c) {
  AttnPattern p;
  p.rows = c->n;
  p.row_offsets.assign(c->row_off, c->row_off + c->n + 1);
  p.cols.assign(c->cols, c->cols + c->nnz);
  return p;
}

Matrix mat(const double* d, int64_t r, int64_t c) {
  Matrix m(r, c);
  if (r * c) std::memcpy(m.data(), d, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

void put(const Matrix& m, double* out) {
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
}

Permutation perm_from(const int64_t* fwd, const int64_t* inv, int64_t n) {
  Permutation p;
  p.forward.assign(fwd, fwd + n);
  p.inverse.assign(inv, inv + n);
  return p;
}

std::vector<WorkerShard> shards_of(int64_t P, int64_t rows, const int64_t* ids, int64_t d,
                                   const double* q, const double* k, const double* v) {
  std::vector<WorkerShard> sh(static_cast<size_t>(P));
  for (int64_t w = 0; w < P; ++w) {
    auto& s = sh[static_cast<size_t>(w)];
    s.worker_id = w;
    s.token_ids.assign(ids + w * rows, ids + (w + 1) * rows);
    s.q_sub = Matrix(rows, d);
    s.k_sub = Matrix(rows, d);
    s.v_sub = Matrix(rows, d);
    for (int64_t r = 0; r < rows; ++r) {
      int64_t t = s.token_ids[static_cast<size_t>(r)];
      std::memcpy(s.q_sub.row(r).data(), q + t * d, sizeof(double) * static_cast<size_t>(d));
      std::memcpy(s.k_sub.row(r).data(), k + t * d, sizeof(double) * static_cast<size_t>(d));
      std::memcpy(s.v_sub.row(r).data(), v + t * d, sizeof(double) * static_cast<size_t>(d));
    }
  }
  return sh;
}

void reassemble(const std::vector<Matrix>& parts, int64_t P, int64_t rows, const int64_t* ids,
                int64_t d, double* out) {
  for (int64_t w = 0; w < P; ++w)
    for (int64_t r = 0; r < rows; ++r)
      std::memcpy(out + ids[w * rows + r] * d, parts[static_cast<size_t>(w)].row(r).data(),
                  sizeof(double) * static_cast<size_t>(d));
}
}  // namespace

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }
void refc_free(void* p) { std::free(p); }

// graph_from_edges (proj/src/graph.cpp:49)
int refc_graph_from_edges(int64_t n, int64_t m, const int64_t* s, const int64_t* d, CCsr* out) {
  return guard([&] {
    std::vector<std::pair<Index, Index>> e(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[static_cast<size_t>(i)] = {s[i], d[i]};
    to_c(graph_from_edges(n, std::move(e)), out);
  });
}

// add_self_loops (proj/src/graph.cpp:127)
int refc_add_self_loops(const CCsr* in, CCsr* out) {
  return guard([&] { to_c(add_self_loops(from_c(in)), out); });
}

// reorder (proj/src/partition.cpp:413)
int refc_reorder(const CCsr* in, int64_t k, uint64_t seed, int64_t* fwd, int64_t* inv) {
  return guard([&] {
    Permutation p = reorder(from_c(in), k, seed);
    std::memcpy(fwd, p.forward.data(), sizeof(int64_t) * p.forward.size());
    std::memcpy(inv, p.inverse.data(), sizeof(int64_t) * p.inverse.size());
  });
}

// permute_graph (proj/src/partition.cpp:435)
int refc_permute_graph(const CCsr* in, const int64_t* fwd, const int64_t* inv, CCsr* out) {
  return guard([&] { to_c(permute_graph(from_c(in), perm_from(fwd, inv, in->n)), out); });
}

// build_cluster_grid (proj/src/partition.cpp:514)
int refc_build_cluster_grid(const CCsr* in, const int64_t* fwd, const int64_t* inv, int64_t k,
                            int64_t* bnd, int64_t* cnnz, double* cden) {
  return guard([&] {
    ClusterGrid g = build_cluster_grid(from_c(in), perm_from(fwd, inv, in->n), k);
    std::memcpy(bnd, g.boundaries.data(), sizeof(int64_t) * g.boundaries.size());
    std::memcpy(cnnz, g.cell_nnz.data(), sizeof(int64_t) * g.cell_nnz.size());
    std::memcpy(cden, g.cell_density.data(), sizeof(double) * g.cell_density.size());
  });
}

// pack_subblocks (proj/src/reformation.cpp:56)
int refc_pack_subblocks(int64_t m, const int64_t* r, const int64_t* c, int64_t nr, int64_t nc,
                        int64_t db, int64_t** tiles, int64_t* nt) {
  return guard([&] {
    std::vector<std::pair<Index, Index>> e(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) e[static_cast<size_t>(i)] = {r[i], c[i]};
    auto t = pack_subblocks(e, nr, nc, db);
    *nt = static_cast<int64_t>(t.size());
    *tiles = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (2 * t.size() + 2)));
    for (size_t i = 0; i < t.size(); ++i) {
      (*tiles)[2 * i] = t[i].row;
      (*tiles)[2 * i + 1] = t[i].col;
    }
  });
}

// build_layout (proj/src/reformation.cpp:111); grid rebuilt from the
// original graph + permutation exactly as callers do.
int refc_build_layout(const CCsr* g_orig, const int64_t* fwd, const int64_t* inv, int64_t k,
                      int strategy, double thre, double bg, int64_t db, int32_t* cell_state,
                      int64_t* block_off, int64_t** blocks, int64_t* dropped, CCsr* pattern) {
  return guard([&] {
    Graph g = from_c(g_orig);
    Permutation p = perm_from(fwd, inv, g_orig->n);
    ClusterGrid grid = build_cluster_grid(g, p, k);
    Graph gp = permute_graph(g, p);
    ClusterSparseLayout L = build_layout(
        grid, gp, strategy == 0 ? TransferStrategy::Indolent : TransferStrategy::Elastic, thre, bg, db);
    std::vector<int64_t> flat;
    block_off[0] = 0;
    for (size_t c = 0; c < L.cell_blocks.size(); ++c) {
      cell_state[c] = L.cell_state[c] == CellState::Transferred ? 1 : 0;
      for (const SubBlock& t : L.cell_blocks[c]) {
        flat.push_back(t.row);
        flat.push_back(t.col);
      }
      block_off[c + 1] = static_cast<int64_t>(flat.size() / 2);
    }
    *blocks = dup_vec(flat);
    *dropped = L.dropped_edges;
    to_c(L.pattern, pattern);
  });
}

// sparse_attention (proj/src/attention.cpp:96)
int refc_sparse_fwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                    const double* v, const CCsr* pat, const double* bias, const double* wm,
                    int forbid, double* out, int64_t* macs) {
  return guard([&] {
    AttnPattern p = pat_from_c(pat);
    std::span<const Real> b, w;
    if (bias) b = {bias, static_cast<size_t>(pat->nnz)};
    if (wm) w = {wm, static_cast<size_t>(pat->nnz)};
    auto r = sparse_attention(mat(q, S, dk), mat(k, S, dk), mat(v, S, dv), p, b, w, forbid != 0);
    put(r.output, out);
    macs[0] = r.macs.score_macs;
    macs[1] = r.macs.weight_macs;
  });
}

// sparse_attention_backward (proj/src/attention.cpp:241)
int refc_sparse_bwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                    const double* v, const CCsr* pat, const double* bias, const double* wm,
                    const double* up, double* dq, double* dkk, double* dvv, double* db) {
  return guard([&] {
    AttnPattern p = pat_from_c(pat);
    std::span<const Real> b, w;
    if (bias) b = {bias, static_cast<size_t>(pat->nnz)};
    if (wm) w = {wm, static_cast<size_t>(pat->nnz)};
    auto g = sparse_attention_backward(mat(q, S, dk), mat(k, S, dk), mat(v, S, dv), p, b, w,
                                       mat(up, S, dv));
    put(g.dq, dq);
    put(g.dk, dkk);
    put(g.dv, dvv);
    if (!g.dbias.empty()) std::memcpy(db, g.dbias.data(), sizeof(double) * g.dbias.size());
  });
}

// dense_attention / dense_attention_backward (proj/src/attention.cpp:46,174)
int refc_dense_fwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                   const double* v, const double* bias, const double* wm, double* out) {
  return guard([&] {
    Matrix B, W;
    if (bias) B = mat(bias, S, S);
    if (wm) W = mat(wm, S, S);
    auto r = dense_attention(mat(q, S, dk), mat(k, S, dk), mat(v, S, dv), bias ? &B : nullptr,
                             wm ? &W : nullptr);
    put(r.output, out);
  });
}

int refc_dense_bwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                   const double* v, const double* bias, const double* wm, const double* up,
                   double* dq, double* dkk, double* dvv, double* db) {
  return guard([&] {
    Matrix B, W;
    if (bias) B = mat(bias, S, S);
    if (wm) W = mat(wm, S, S);
    auto g = dense_attention_backward(mat(q, S, dk), mat(k, S, dk), mat(v, S, dv),
                                      bias ? &B : nullptr, wm ? &W : nullptr, mat(up, S, dv));
    put(g.dq, dq);
    put(g.dk, dkk);
    put(g.dv, dvv);
    std::memcpy(db, g.dbias.data(), sizeof(double) * g.dbias.size());
  });
}

// partition_sequence (proj/src/parallel.cpp:96)
int refc_partition_sequence(int64_t S, int64_t P, uint64_t seed, int64_t* ids) {
  return guard([&] {
    auto sh = partition_sequence(S, P, seed);
    size_t o = 0;
    for (auto& s : sh)
      for (Index t : s.token_ids) ids[o++] = t;
  });
}

// run_distributed_layer (proj/src/parallel.cpp:190); shards assembled from
// token-indexed full matrices with the given ids.
int refc_dist_fwd(int64_t P, int64_t S, int64_t d, int64_t H, const int64_t* ids,
                  const double* q, const double* k, const double* v, const CCsr* pat,
                  const int64_t* fwd, const int64_t* inv, const double* bias, const double* wm,
                  double* out, int64_t* ledger, int64_t* macs) {
  return guard([&] {
    const int64_t rows = S / P;
    auto sh = shards_of(P, rows, ids, d, q, k, v);
    CommLedger L(P);
    std::span<const Real> b, w;
    if (bias) b = {bias, static_cast<size_t>(pat->nnz)};
    if (wm) w = {wm, static_cast<size_t>(H * pat->nnz)};
    auto r = run_distributed_layer(sh, pat_from_c(pat), perm_from(fwd, inv, S), H, b, w, L);
    reassemble(r.out_shards, P, rows, ids, d, out);
    for (int64_t i = 0; i < P; ++i) {
      auto& e = L.workers[static_cast<size_t>(i)];
      ledger[i * 5 + 0] = e.qkv_gather;
      ledger[i * 5 + 1] = e.qkv_gather_cross;
      ledger[i * 5 + 2] = e.output_scatter;
      ledger[i * 5 + 3] = e.output_scatter_cross;
      ledger[i * 5 + 4] = e.bias_exchange;
    }
    *macs = r.macs.score_macs;
  });
}

// run_distributed_layer_backward (proj/src/parallel.cpp:271)
int refc_dist_bwd(int64_t P, int64_t S, int64_t d, int64_t H, const int64_t* ids,
                  const double* q, const double* k, const double* v, const CCsr* pat,
                  const int64_t* fwd, const int64_t* inv, const double* bias, const double* wm,
                  const double* up, double* dq, double* dkk, double* dvv, double* dbias) {
  return guard([&] {
    const int64_t rows = S / P;
    auto sh = shards_of(P, rows, ids, d, q, k, v);
    std::vector<Matrix> ups;
    for (int64_t w = 0; w < P; ++w) {
      Matrix u(rows, d);
      for (int64_t r = 0; r < rows; ++r)
        std::memcpy(u.row(r).data(), up + ids[w * rows + r] * d, sizeof(double) * static_cast<size_t>(d));
      ups.push_back(std::move(u));
    }
    std::span<const Real> b, w;
    if (bias) b = {bias, static_cast<size_t>(pat->nnz)};
    if (wm) w = {wm, static_cast<size_t>(H * pat->nnz)};
    auto g = run_distributed_layer_backward(sh, pat_from_c(pat), perm_from(fwd, inv, S), H, b, w, ups);
    reassemble(g.dq_sub, P, rows, ids, d, dq);
    reassemble(g.dk_sub, P, rows, ids, d, dkk);
    reassemble(g.dv_sub, P, rows, ids, d, dvv);
    std::memcpy(dbias, g.dbias.data(), sizeof(double) * g.dbias.size());
  });
}

// check_conditions (proj/src/interleave.cpp:68)
int refc_check_conditions(const CCsr* g, int64_t layers, int32_t* flags, int64_t* ints) {
  return guard([&] {
    ConditionReport r = check_conditions(from_c(g), layers);
    flags[0] = r.c1_self_attend;
    flags[1] = r.c2_hamiltonian == HamiltonianCheck::Pass;
    flags[2] = r.c3_reachable_within_l;
    ints[0] = r.layers;
    ints[1] = r.sweep_from;
    ints[2] = r.sweep_to;
    ints[3] = r.diameter_lower_bound;
  });
}

// generate_sbm (proj/src/model.cpp:187) — fixture source for partition tests
int refc_generate_sbm(int64_t n, int64_t blocks, double pin, double pout, uint64_t seed,
                      double noise, CCsr* out, int32_t* labels) {
  return guard([&] {
    Graph g = generate_sbm(n, blocks, pin, pout, seed, noise);
    to_c(g, out);
    for (int64_t i = 0; i < n; ++i) labels[i] = g.labels[static_cast<size_t>(i)];
  });
}

// oracle::random_graph (proj/tests/oracles.hpp:71)
int refc_random_graph(int64_t n, double p, uint64_t seed, int loops, CCsr* out) {
  return guard([&] { to_c(oracle::random_graph(n, p, seed, loops != 0), out); });
}

// Matrix::randn (proj/src/matrix.cpp) — so fixtures can reproduce the
// reference tests' inputs draw for draw.
int refc_randn_sequence(uint64_t seed, int64_t count, const int64_t* rows, const int64_t* cols,
                        const double* std_, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    size_t o = 0;
    for (int64_t i = 0; i < count; ++i) {
      Matrix m = Matrix::randn(rows[i], cols[i], std_[i], rng);
      std::memcpy(out + o, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
      o += static_cast<size_t>(m.size());
    }
  });
}

// make_tuner_state + tuner_update (proj/src/reformation.cpp:224-265)
int refc_tuner_run(double bg, int64_t delta, int64_t n, const double* loss, const double* et,
                   int64_t* idx, double* avg, double* thr, int64_t* nthr) {
  return guard([&] {
    TunerState st = make_tuner_state(bg, delta);
    *nthr = static_cast<int64_t>(st.thresholds.size());
    for (size_t i = 0; i < st.thresholds.size(); ++i) thr[i] = st.thresholds[i];
    for (int64_t e = 0; e < n; ++e) {
      tuner_update(st, loss[e], et[e], e);
      idx[e] = static_cast<int64_t>(st.idx);
      avg[e] = st.avg_loss;
    }
  });
}

int refc_select_k(int64_t l2, int64_t d, int64_t i, int64_t* out) {
  return guard([&] { *out = select_k(l2, d, i); });
}

int refc_select_db(int64_t n, const int64_t* db, const double* thr, int64_t* out) {
  return guard([&] {
    std::map<Index, Real> prof;
    for (int64_t i = 0; i < n; ++i) prof[db[i]] = thr[i];
    *out = select_db(prof);
  });
}


// gte::spd_table (proj/src/graph.cpp:216-262): malloc-owned CSR + distances
int refc_spd_table(const CCsr* g, int64_t max_dist, int64_t** row_off, int64_t** cols, uint16_t** dist,
                   int64_t* nnz) {
  return guard([&] {
    Graph gr = from_c(g);
    SpdTable t = spd_table(gr, static_cast<int>(max_dist));
    *nnz = static_cast<int64_t>(t.cols.size());
    *row_off = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * t.row_offsets.size()));
    *cols = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (t.cols.size() + 1)));
    *dist = static_cast<uint16_t*>(std::malloc(sizeof(uint16_t) * (t.dist.size() + 1)));
    std::memcpy(*row_off, t.row_offsets.data(), sizeof(int64_t) * t.row_offsets.size());
    std::memcpy(*cols, t.cols.data(), sizeof(int64_t) * t.cols.size());
    std::memcpy(*dist, t.dist.data(), sizeof(uint16_t) * t.dist.size());
  });
}

}  // extern "C"

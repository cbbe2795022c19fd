/* TEST INFRASTRUCTURE — not product code. CPU oracle, see oracle.h.
 * Elastic Computation Reformation restated from
 *   /root/reference/proj/src/reformation.cpp:12-296 (packing, layout, tuner)
 * and the interleave policy from /root/reference/proj/src/interleave.cpp:10-106.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

int orc_fail(int code, const char* fmt, ...);

static inline int64_t i64abs(int64_t x) { return x < 0 ? -x : x; }

/* packer used by orc_build_layout: 0 auto (the field restatement below for
 * cells up to 2^24 positions, the candidate-origin restatement of
 * orc_pack_sparse.cpp above), 1 always the field, 2 always candidates */
static int g_pack_mode = 0;
void orc_set_pack_mode(int mode) { g_pack_mode = mode; }

/* pack_subblocks: greedy max-cover of not-yet-covered edges with non-overlapping
 * d_b x d_b tiles; ties keep the first (raster-order) origin; stops only if no
 * free origin remains. reformation.cpp:56-109 (prefix field :15-37). */
int orc_pack_subblocks(int64_t m, const int64_t* er, const int64_t* ec, int64_t n_rows,
                       int64_t n_cols, int64_t d_b, int64_t* tiles_rc, int64_t cap,
                       int64_t* ntiles) {
  *ntiles = 0;
  if (d_b < 1) return orc_fail(ORC_CONFIG, "pack_subblocks: d_b must be >= 1");
  if (d_b > n_rows || d_b > n_cols)
    return orc_fail(ORC_CONFIG, "pack_subblocks: d_b %lld too large for %lldx%lld cell",
                    (long long)d_b, (long long)n_rows, (long long)n_cols);
  if (m == 0) return ORC_OK;
  int32_t* grid = (int32_t*)calloc((size_t)(n_rows * n_cols), sizeof(int32_t));
  for (int64_t e = 0; e < m; ++e) {
    if (er[e] < 0 || er[e] >= n_rows || ec[e] < 0 || ec[e] >= n_cols) {
      free(grid);
      return orc_fail(ORC_CONFIG, "pack_subblocks: edge outside cell");
    }
    grid[er[e] * n_cols + ec[e]] = 1;
  }
  const int64_t want = (m + d_b * d_b - 1) / (d_b * d_b);
  const int64_t W = n_cols + 1;
  int64_t* pre = (int64_t*)malloc(sizeof(int64_t) * (size_t)((n_rows + 1) * W));
  int64_t nt = 0;
  while (nt < want) {
    memset(pre, 0, sizeof(int64_t) * (size_t)((n_rows + 1) * W));
    for (int64_t i = 0; i < n_rows; ++i)
      for (int64_t j = 0; j < n_cols; ++j)
        pre[(i + 1) * W + j + 1] = pre[i * W + j + 1] + pre[(i + 1) * W + j] - pre[i * W + j] +
                                   grid[i * n_cols + j];
    int64_t br = -1, bc = -1, best = -1;
    for (int64_t r = 0; r + d_b <= n_rows; ++r) {
      for (int64_t c = 0; c + d_b <= n_cols; ++c) {
        int clash = 0;
        for (int64_t t = 0; t < nt; ++t) {
          if (i64abs(r - tiles_rc[2 * t]) < d_b && i64abs(c - tiles_rc[2 * t + 1]) < d_b) {
            clash = 1;
            break;
          }
        }
        if (clash) continue;
        int64_t cover = pre[(r + d_b) * W + c + d_b] - pre[r * W + c + d_b] -
                        pre[(r + d_b) * W + c] + pre[r * W + c];
        if (cover > best) {
          best = cover;
          br = r;
          bc = c;
        }
      }
    }
    if (best < 0) break;
    if (nt >= cap) {
      free(pre);
      free(grid);
      return orc_fail(ORC_CONFIG, "pack_subblocks: tile buffer too small");
    }
    tiles_rc[2 * nt] = br;
    tiles_rc[2 * nt + 1] = bc;
    ++nt;
    for (int64_t r = br; r < br + d_b; ++r)
      for (int64_t c = bc; c < bc + d_b; ++c) grid[r * n_cols + c] = 0;
  }
  *ntiles = nt;
  free(pre);
  free(grid);
  return ORC_OK;
}

void orc_layout_free(orc_layout* L) {
  if (!L) return;
  free(L->boundaries);
  free(L->cell_state);
  free(L->block_off);
  free(L->blocks);
  orc_csr_free(&L->pattern);
  memset(L, 0, sizeof *L);
}

typedef struct {
  int64_t* r;
  int64_t* c;
  int64_t n, cap;
} evec;

static void evec_push(evec* v, int64_t r, int64_t c) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 16;
    v->r = (int64_t*)realloc(v->r, sizeof(int64_t) * (size_t)v->cap);
    v->c = (int64_t*)realloc(v->c, sizeof(int64_t) * (size_t)v->cap);
  }
  v->r[v->n] = r;
  v->c[v->n] = c;
  v->n++;
}

typedef struct {
  int64_t a, b;
} span2;

static int cmp_span(const void* x, const void* y) {
  const span2* p = (const span2*)x;
  const span2* q = (const span2*)y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return 0;
}

/* build_layout: classify (Transferred iff cell_density < threshold), pack,
 * count drops, materialise the sorted pattern. reformation.cpp:111-195 */
int orc_build_layout(int64_t k, const int64_t* bnd, const int64_t* cell_nnz,
                     const double* cell_density, const orc_csr* g, int strategy,
                     double beta_thre, double beta_g, int64_t d_b, orc_layout* L) {
  memset(L, 0, sizeof *L);
  const int64_t n = g->n;
  if (bnd[k] != n) return orc_fail(ORC_CONFIG, "build_layout: grid/graph size mismatch");
  int64_t tot = 0;
  for (int64_t c = 0; c < k * k; ++c) tot += cell_nnz[c];
  if (tot != g->nnz) return orc_fail(ORC_CONFIG, "build_layout: grid/graph nnz mismatch");
  const double threshold = strategy == 0 ? beta_g : beta_thre;
  L->seq_len = n;
  L->k = k;
  L->d_b = d_b;
  L->boundaries = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
  memcpy(L->boundaries, bnd, sizeof(int64_t) * (size_t)(k + 1));
  L->cell_state = (int32_t*)calloc((size_t)(k * k), sizeof(int32_t));
  L->block_off = (int64_t*)calloc((size_t)(k * k + 1), sizeof(int64_t));
  evec* cells = (evec*)calloc((size_t)(k * k), sizeof(evec));
  for (int64_t u = 0; u < n; ++u) {
    int64_t a = orc_cluster_of(n, k, u);
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      int64_t v = g->cols[e];
      int64_t b = orc_cluster_of(n, k, v);
      evec_push(&cells[a * k + b], u - bnd[a], v - bnd[b]);
    }
  }
  int64_t** tiles = (int64_t**)calloc((size_t)(k * k), sizeof(int64_t*));
  int64_t* ntile = (int64_t*)calloc((size_t)(k * k), sizeof(int64_t));
  int rc = ORC_OK;
  for (int64_t a = 0; a < k && rc == ORC_OK; ++a) {
    for (int64_t b = 0; b < k; ++b) {
      int64_t cell = a * k + b;
      if (cell_density[cell] >= threshold) continue;
      L->cell_state[cell] = 1;
      if (cells[cell].n == 0) continue;
      int64_t cap = (cells[cell].n + d_b * d_b - 1) / (d_b * d_b);
      tiles[cell] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * cap + 2));
      const int64_t nr = bnd[a + 1] - bnd[a], nc = bnd[b + 1] - bnd[b];
      const int sparse = g_pack_mode == 2 || (g_pack_mode == 0 && nr * nc > ((int64_t)1 << 24));
      rc = (sparse ? orc_pack_subblocks_sparse : orc_pack_subblocks)(cells[cell].n, cells[cell].r, cells[cell].c,
                                                                     nr, nc, d_b, tiles[cell], cap, &ntile[cell]);
      if (rc) break;
      int64_t covered = 0;
      for (int64_t e = 0; e < cells[cell].n; ++e) {
        int64_t r = cells[cell].r[e], c = cells[cell].c[e];
        for (int64_t t = 0; t < ntile[cell]; ++t) {
          int64_t tr = tiles[cell][2 * t], tc = tiles[cell][2 * t + 1];
          if (r >= tr && r < tr + d_b && c >= tc && c < tc + d_b) {
            ++covered;
            break;
          }
        }
      }
      L->dropped_edges += cells[cell].n - covered;
    }
  }
  if (rc == ORC_OK) {
    for (int64_t c = 0; c < k * k; ++c) L->block_off[c + 1] = L->block_off[c] + ntile[c];
    L->blocks = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * L->block_off[k * k] + 2));
    for (int64_t c = 0; c < k * k; ++c)
      if (ntile[c])
        memcpy(L->blocks + 2 * L->block_off[c], tiles[c], sizeof(int64_t) * (size_t)(2 * ntile[c]));
    /* materialise: count first, then fill */
    int64_t total = 0;
    L->pattern.n = n;
    L->pattern.row_off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t maxt = 1;
    for (int64_t c = 0; c < k * k; ++c)
      if (ntile[c] > maxt) maxt = ntile[c];
    span2* spans = (span2*)malloc(sizeof(span2) * (size_t)maxt);
    for (int pass = 0; pass < 2; ++pass) {
      int64_t w = 0;
      for (int64_t u = 0; u < n; ++u) {
        int64_t a = orc_cluster_of(n, k, u);
        int64_t lr = u - bnd[a];
        for (int64_t b = 0; b < k; ++b) {
          int64_t cell = a * k + b;
          if (L->cell_state[cell] == 0) {
            for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
              int64_t v = g->cols[e];
              if (v >= bnd[b] && v < bnd[b + 1]) {
                if (pass) L->pattern.cols[w] = v;
                ++w;
              }
            }
          } else {
            int64_t ns = 0;
            for (int64_t t = 0; t < ntile[cell]; ++t) {
              int64_t tr = tiles[cell][2 * t], tc = tiles[cell][2 * t + 1];
              if (lr >= tr && lr < tr + d_b) {
                spans[ns].a = tc;
                spans[ns].b = tc + d_b;
                ++ns;
              }
            }
            qsort(spans, (size_t)ns, sizeof(span2), cmp_span);
            for (int64_t s = 0; s < ns; ++s)
              for (int64_t c = spans[s].a; c < spans[s].b; ++c) {
                if (pass) L->pattern.cols[w] = bnd[b] + c;
                ++w;
              }
          }
        }
        if (pass) L->pattern.row_off[u + 1] = w;
      }
      if (!pass) {
        total = w;
        L->pattern.cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 1));
      }
    }
    L->pattern.nnz = total;
    free(spans);
  }
  for (int64_t c = 0; c < k * k; ++c) {
    free(cells[c].r);
    free(cells[c].c);
    free(tiles[c]);
  }
  free(cells);
  free(tiles);
  free(ntile);
  if (rc) orc_layout_free(L);
  return rc;
}

static int cmp_dbl(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* make_tuner_state: reformation.cpp:224-238 */
int orc_make_tuner(double beta_g, int64_t delta, orc_tuner* st) {
  memset(st, 0, sizeof *st);
  if (beta_g < 0.0 || beta_g > 1.0) return orc_fail(ORC_CONFIG, "tuner: beta_g must lie in [0, 1]");
  if (delta < 1) return orc_fail(ORC_CONFIG, "tuner: delta must be >= 1");
  st->delta = delta;
  double raw[7] = {0.0, beta_g, 1.5 * beta_g, 5.0 * beta_g, 7.0 * beta_g, 10.0 * beta_g, 1.0};
  for (int i = 0; i < 7; ++i)
    if (raw[i] > 1.0) raw[i] = 1.0;
  qsort(raw, 7, sizeof(double), cmp_dbl);
  int64_t n = 0;
  for (int i = 0; i < 7; ++i)
    if (n == 0 || raw[i] != st->thresholds[n - 1]) st->thresholds[n++] = raw[i];
  st->n_thr = n;
  double key = beta_g < 1.0 ? beta_g : 1.0;
  int64_t idx = 0;
  while (idx < n && st->thresholds[idx] < key) ++idx;
  st->idx = idx;
  return ORC_OK;
}

void orc_tuner_free(orc_tuner* st) {
  free(st->ldr_epoch);
  free(st->ldr_val);
  st->ldr_epoch = NULL;
  st->ldr_val = NULL;
}

static void push_ldr(orc_tuner* st, int64_t e, double v) {
  if (st->n_ldr == st->cap_ldr) {
    st->cap_ldr = st->cap_ldr ? 2 * st->cap_ldr : 16;
    st->ldr_epoch = (int64_t*)realloc(st->ldr_epoch, sizeof(int64_t) * (size_t)st->cap_ldr);
    st->ldr_val = (double*)realloc(st->ldr_val, sizeof(double) * (size_t)st->cap_ldr);
  }
  st->ldr_epoch[st->n_ldr] = e;
  st->ldr_val[st->n_ldr] = v;
  st->n_ldr++;
}

/* tuner_update: reformation.cpp:240-265 */
int orc_tuner_update(orc_tuner* st, double loss, double et, int64_t epoch) {
  if (et <= 0.0) return orc_fail(ORC_CONFIG, "tuner_update: epoch_time must be positive");
  if (!st->has_loss) {
    st->avg_loss = loss;
    st->has_loss = 1;
    push_ldr(st, epoch, 0.0);
    return ORC_OK;
  }
  if (st->n_ldr > 0 && epoch != st->ldr_epoch[st->n_ldr - 1] + 1)
    return orc_fail(ORC_CONFIG, "tuner_update: epochs must be consecutive");
  const double prev = st->avg_loss;
  st->avg_loss = 0.9 * prev + 0.1 * loss;
  const double ldr = (st->avg_loss - prev) / et;
  push_ldr(st, epoch, ldr);
  const int64_t lag = st->n_ldr - 1 - st->delta;
  if (epoch >= st->delta && lag >= 0) {
    if (ldr >= st->ldr_val[lag]) {
      if (st->idx + 1 < st->n_thr) st->idx++;
    } else if (st->idx > 0) {
      st->idx--;
    }
  }
  return ORC_OK;
}

/* select_k: bit_floor(floor(sqrt(l2 / (i * d)))). reformation.cpp:267-275 */
int orc_select_k(int64_t l2_bytes, int64_t hidden_dim, int64_t i, int64_t* out) {
  if (l2_bytes <= 0 || hidden_dim <= 0 || i <= 0)
    return orc_fail(ORC_CONFIG, "select_k: all arguments must be positive");
  double raw = floor(sqrt((double)l2_bytes / ((double)i * (double)hidden_dim)));
  if (raw < 1.0) return orc_fail(ORC_CONFIG, "select_k: cache budget yields k < 1");
  uint64_t r = (uint64_t)raw, p = 1;
  while (p <= r / 2) p <<= 1;
  *out = (int64_t)p;
  return ORC_OK;
}

/* select_db: argmax, ties toward the median position (larger d_b on equal
 * distance). Entries ascending by d_b (std::map order). reformation.cpp:277-296 */
int orc_select_db(int64_t n, const int64_t* db, const double* thr, int64_t* out) {
  if (n == 0) return orc_fail(ORC_CONFIG, "select_db: empty profile");
  double best = -INFINITY;
  for (int64_t i = 0; i < n; ++i)
    if (thr[i] > best) best = thr[i];
  const double median = (double)(n - 1) / 2.0;
  int64_t chosen = -1;
  double cd = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (thr[i] != best) continue;
    double dist = fabs((double)i - median);
    if (chosen == -1 || dist < cd || (dist == cd && db[i] > chosen)) {
      chosen = db[i];
      cd = dist;
    }
  }
  *out = chosen;
  return ORC_OK;
}

/* ---- interleave: proj/src/interleave.cpp ---- */

typedef struct {
  int64_t* off;
  int64_t* adj;
  int64_t n;
} sadj;

static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* sym_adj_no_loops: interleave.cpp:39-53 */
static void sym_adj(const orc_csr* g, sadj* s) {
  int64_t n = g->n;
  int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      int64_t v = g->cols[e];
      if (u == v) continue;
      deg[u]++;
      deg[v]++;
    }
  int64_t* off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t u = 0; u < n; ++u) off[u + 1] = off[u] + deg[u];
  int64_t* adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(off[n] + 1));
  int64_t* fill = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      int64_t v = g->cols[e];
      if (u == v) continue;
      adj[off[u] + fill[u]++] = v;
      adj[off[v] + fill[v]++] = u;
    }
  /* sort + unique per node, compacting */
  int64_t* noff = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t w = 0;
  for (int64_t u = 0; u < n; ++u) {
    int64_t b = off[u], e1 = off[u + 1];
    qsort(adj + b, (size_t)(e1 - b), sizeof(int64_t), cmp_i64);
    for (int64_t e = b; e < e1; ++e)
      if (e == b || adj[e] != adj[e - 1]) adj[w++] = adj[e];
    noff[u + 1] = w;
  }
  free(deg);
  free(off);
  free(fill);
  s->off = noff;
  s->adj = adj;
  s->n = n;
}

/* bfs_farthest: interleave.cpp:12-37 */
static int64_t bfs_far(const sadj* s, int64_t src, int* dist) {
  for (int64_t i = 0; i < s->n; ++i) dist[i] = -1;
  int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->n + 1));
  int64_t* nx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->n + 1));
  int64_t nf = 1;
  fr[0] = src;
  dist[src] = 0;
  int64_t far = src;
  int far_d = 0;
  while (nf) {
    int64_t nn = 0;
    for (int64_t a = 0; a < nf; ++a) {
      int64_t u = fr[a];
      for (int64_t e = s->off[u]; e < s->off[u + 1]; ++e) {
        int64_t v = s->adj[e];
        if (dist[v] == -1) {
          dist[v] = dist[u] + 1;
          nx[nn++] = v;
          if (dist[v] > far_d || (dist[v] == far_d && v < far)) {
            far_d = dist[v];
            far = v;
          }
        }
      }
    }
    int64_t* t = fr; fr = nx; nx = t;
    nf = nn;
  }
  free(fr);
  free(nx);
  return far;
}

/* check_conditions: interleave.cpp:68-99 */
int orc_check_conditions(const orc_csr* g, int64_t layers, orc_conditions* r) {
  memset(r, 0, sizeof *r);
  r->layers = layers;
  r->sweep_from = r->sweep_to = r->diameter_lower_bound = -1;
  const int64_t n = g->n;
  r->c1_self_attend = 1;
  for (int64_t u = 0; u < n && r->c1_self_attend; ++u) {
    int found = 0;
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e)
      if (g->cols[e] == u) found = 1;
    if (!found) r->c1_self_attend = 0;
  }
  sadj s;
  sym_adj(g, &s);
  int64_t min_deg = n == 0 ? 0 : s.off[1] - s.off[0];
  for (int64_t u = 0; u < n; ++u)
    if (s.off[u + 1] - s.off[u] < min_deg) min_deg = s.off[u + 1] - s.off[u];
  r->c2_pass = (n >= 1 && 2 * min_deg >= n) ? 1 : 0;
  if (n >= 1) {
    int* dist = (int*)malloc(sizeof(int) * (size_t)n);
    int64_t u = bfs_far(&s, 0, dist);
    int connected = 1;
    for (int64_t i = 0; i < n; ++i)
      if (dist[i] == -1) connected = 0;
    int64_t v = bfs_far(&s, u, dist);
    r->sweep_from = u;
    r->sweep_to = v;
    r->diameter_lower_bound = dist[v];
    r->c3_reachable_within_l = connected && r->diameter_lower_bound <= layers;
    free(dist);
  }
  free(s.off);
  free(s.adj);
  return ORC_OK;
}

/* select_mode: interleave.cpp:101-106 */
int orc_select_mode(const orc_conditions* r, int64_t epoch, int64_t period, int32_t* mode,
                    int32_t* reason) {
  if (period < 1) return orc_fail(ORC_CONFIG, "select_mode: dense_period must be >= 1");
  if (epoch % period == 0) {
    *mode = 1;
    *reason = 1;
  } else if (!(r->c1_self_attend && r->c2_pass && r->c3_reachable_within_l)) {
    *mode = 1;
    *reason = 0;
  } else {
    *mode = 0;
    *reason = 2;
  }
  return ORC_OK;
}

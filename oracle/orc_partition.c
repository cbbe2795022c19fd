/* TEST INFRASTRUCTURE — not product code. CPU oracle, see oracle.h.
 * Faithful (deliberately naive, O(n^2) scans kept) restatement of the
 * reference multilevel recursive bisection and the k x k cluster grid:
 *   /root/reference/proj/src/partition.cpp:15-547.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "orc_rng.h"

int orc_fail(int code, const char* fmt, ...);

#define MAX_FM_PASSES 10   /* partition.cpp:17 */
#define BALANCE_TOL 0.05   /* partition.cpp:18 */

typedef struct {
  int64_t n;
  int64_t* off;  /* n+1 */
  int64_t* adj;
  int64_t* ew;
  int64_t* nw;   /* n */
  int64_t m;     /* arcs */
} ugraph;

static void ug_free(ugraph* g) {
  free(g->off);
  free(g->adj);
  free(g->ew);
  free(g->nw);
  memset(g, 0, sizeof *g);
}

static int64_t ug_total_weight(const ugraph* g) {
  int64_t s = 0;
  for (int64_t i = 0; i < g->n; ++i) s += g->nw[i];
  return s;
}

typedef struct {
  int64_t u, v;
} p2;

static int cmp_p2(const void* a, const void* b) {
  const p2* x = (const p2*)a;
  const p2* y = (const p2*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}

/* ugraph_from: drop loops, add both arc directions, sort, merge duplicates
 * into weights. partition.cpp:40-66 */
static void ugraph_from(const orc_csr* g, ugraph* ug) {
  p2* und = (p2*)malloc(sizeof(p2) * (size_t)(2 * g->nnz + 1));
  int64_t m = 0;
  for (int64_t u = 0; u < g->n; ++u) {
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      int64_t v = g->cols[e];
      if (u == v) continue;
      und[m].u = u; und[m].v = v; ++m;
      und[m].u = v; und[m].v = u; ++m;
    }
  }
  qsort(und, (size_t)m, sizeof(p2), cmp_p2);
  ug->n = g->n;
  ug->off = (int64_t*)calloc((size_t)g->n + 1, sizeof(int64_t));
  ug->nw = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n + 1));
  for (int64_t i = 0; i < g->n; ++i) ug->nw[i] = 1;
  ug->adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  ug->ew = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t w = 0;
  for (int64_t i = 0; i < m;) {
    int64_t j = i;
    while (j < m && und[j].u == und[i].u && und[j].v == und[i].v) ++j;
    ug->adj[w] = und[i].v;
    ug->ew[w] = j - i;
    ++w;
    ug->off[und[i].u + 1] = w;
    i = j;
  }
  for (int64_t u = 0; u < ug->n; ++u)
    if (ug->off[u + 1] < ug->off[u]) ug->off[u + 1] = ug->off[u];
  ug->m = w;
  free(und);
}

typedef struct {
  int64_t u, v, w;
} p3;

static int cmp_p3(const void* a, const void* b) {
  const p3* x = (const p3*)a;
  const p3* y = (const p3*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  if (x->w != y->w) return x->w < y->w ? -1 : 1;
  return 0;
}

/* contract: partition.cpp:73-109 */
static void contract(const ugraph* ug, const int64_t* partner, ugraph* coarse, int64_t* f2c) {
  for (int64_t u = 0; u < ug->n; ++u) f2c[u] = -1;
  int64_t next = 0;
  for (int64_t u = 0; u < ug->n; ++u) {
    if (f2c[u] != -1) continue;
    f2c[u] = next;
    if (partner[u] != u) f2c[partner[u]] = next;
    ++next;
  }
  coarse->n = next;
  coarse->nw = (int64_t*)calloc((size_t)next + 1, sizeof(int64_t));
  for (int64_t u = 0; u < ug->n; ++u) coarse->nw[f2c[u]] += ug->nw[u];
  p3* ed = (p3*)malloc(sizeof(p3) * (size_t)(ug->m + 1));
  int64_t m = 0;
  for (int64_t u = 0; u < ug->n; ++u) {
    int64_t cu = f2c[u];
    for (int64_t e = ug->off[u]; e < ug->off[u + 1]; ++e) {
      int64_t cv = f2c[ug->adj[e]];
      if (cu == cv) continue;
      ed[m].u = cu; ed[m].v = cv; ed[m].w = ug->ew[e]; ++m;
    }
  }
  qsort(ed, (size_t)m, sizeof(p3), cmp_p3);
  coarse->off = (int64_t*)calloc((size_t)next + 1, sizeof(int64_t));
  coarse->adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  coarse->ew = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t w = 0;
  for (int64_t i = 0; i < m;) {
    int64_t j = i, s = 0;
    while (j < m && ed[j].u == ed[i].u && ed[j].v == ed[i].v) s += ed[j++].w;
    coarse->adj[w] = ed[i].v;
    coarse->ew[w] = s;
    ++w;
    coarse->off[ed[i].u + 1] = w;
    i = j;
  }
  for (int64_t u = 0; u < next; ++u)
    if (coarse->off[u + 1] < coarse->off[u]) coarse->off[u + 1] = coarse->off[u];
  coarse->m = w;
  free(ed);
}

/* heavy_edge_matching: partition.cpp:111-138 */
static void heavy_edge_matching(const ugraph* ug, orc_mt64* rng, int64_t* partner) {
  int64_t n = ug->n;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  orc_shuffle_i64(order, n, rng);
  for (int64_t i = 0; i < n; ++i) partner[i] = i;
  char* matched = (char*)calloc((size_t)n + 1, 1);
  for (int64_t oi = 0; oi < n; ++oi) {
    int64_t u = order[oi];
    if (matched[u]) continue;
    int64_t best = -1, best_w = -1;
    for (int64_t e = ug->off[u]; e < ug->off[u + 1]; ++e) {
      int64_t v = ug->adj[e];
      if (matched[v] || v == u) continue;
      if (ug->ew[e] > best_w || (ug->ew[e] == best_w && v < best)) {
        best_w = ug->ew[e];
        best = v;
      }
    }
    if (best != -1) {
      matched[u] = matched[best] = 1;
      partner[u] = best;
      partner[best] = u;
    }
  }
  free(order);
  free(matched);
}

/* farthest_from: BFS, max depth, smallest id among ties. partition.cpp:142-166 */
static int64_t farthest_from(const ugraph* ug, int64_t src, int* dist) {
  for (int64_t i = 0; i < ug->n; ++i) dist[i] = -1;
  int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ug->n + 1));
  int64_t* nx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ug->n + 1));
  int64_t nf = 1, nn;
  fr[0] = src;
  dist[src] = 0;
  int64_t far = src;
  int far_d = 0;
  while (nf > 0) {
    nn = 0;
    for (int64_t a = 0; a < nf; ++a) {
      int64_t u = fr[a];
      for (int64_t e = ug->off[u]; e < ug->off[u + 1]; ++e) {
        int64_t v = ug->adj[e];
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

/* cut_weight: partition.cpp:168-176 */
static int64_t cut_weight(const ugraph* ug, const int* side) {
  int64_t cut = 0;
  for (int64_t u = 0; u < ug->n; ++u)
    for (int64_t e = ug->off[u]; e < ug->off[u + 1]; ++e)
      if (side[u] != side[ug->adj[e]]) cut += ug->ew[e];
  return cut / 2;
}

/* balance_allowance: partition.cpp:178-184 */
static int64_t balance_allowance(const ugraph* ug) {
  int64_t max_nw = 1;
  if (ug->n > 0) {
    max_nw = ug->nw[0];
    for (int64_t i = 1; i < ug->n; ++i)
      if (ug->nw[i] > max_nw) max_nw = ug->nw[i];
  }
  int64_t a = (int64_t)(2 * BALANCE_TOL * (double)ug_total_weight(ug));
  return a > 2 * max_nw ? a : 2 * max_nw;
}

static inline int64_t i64abs(int64_t x) { return x < 0 ? -x : x; }

/* fm_refine: classic FM with best-prefix rollback. partition.cpp:187-245 */
static void fm_refine(const ugraph* ug, int* side, int64_t allow) {
  const int64_t n = ug->n;
  int64_t side_w[2] = {0, 0};
  for (int64_t v = 0; v < n; ++v) side_w[side[v]] += ug->nw[v];
  int64_t* gain = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  char* locked = (char*)malloc((size_t)n + 1);
  int64_t* moves = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int pass = 0; pass < MAX_FM_PASSES; ++pass) {
    for (int64_t v = 0; v < n; ++v) {
      int64_t g = 0;
      for (int64_t e = ug->off[v]; e < ug->off[v + 1]; ++e)
        g += (side[ug->adj[e]] != side[v]) ? ug->ew[e] : -ug->ew[e];
      gain[v] = g;
      locked[v] = 0;
    }
    int64_t nmoves = 0, cum = 0, best_cum = 0, best_prefix = 0;
    for (;;) {
      int64_t best = -1;
      for (int64_t v = 0; v < n; ++v) {
        if (locked[v]) continue;
        int from = side[v];
        int64_t imb = i64abs((side_w[from] - ug->nw[v]) - (side_w[1 - from] + ug->nw[v]));
        if (imb > allow) continue;
        if (best == -1 || gain[v] > gain[best] || (gain[v] == gain[best] && v < best)) best = v;
      }
      if (best == -1) break;
      int from = side[best];
      side[best] = 1 - from;
      side_w[from] -= ug->nw[best];
      side_w[1 - from] += ug->nw[best];
      locked[best] = 1;
      cum += gain[best];
      moves[nmoves++] = best;
      for (int64_t e = ug->off[best]; e < ug->off[best + 1]; ++e) {
        int64_t nb = ug->adj[e];
        if (locked[nb]) continue;
        gain[nb] += (side[nb] == side[best]) ? -2 * ug->ew[e] : 2 * ug->ew[e];
      }
      if (cum > best_cum) {
        best_cum = cum;
        best_prefix = nmoves;
      }
    }
    for (int64_t i = nmoves; i > best_prefix; --i) {
      int64_t v = moves[i - 1];
      int from = side[v];
      side[v] = 1 - from;
      side_w[from] -= ug->nw[v];
      side_w[1 - from] += ug->nw[v];
    }
    if (best_cum <= 0) break;
  }
  free(gain);
  free(locked);
  free(moves);
}

/* grow_region: partition.cpp:248-277 */
static void grow_region(const ugraph* ug, int64_t seed, int* side) {
  const int64_t n = ug->n;
  for (int64_t i = 0; i < n; ++i) side[i] = 1;
  const int64_t target = ug_total_weight(ug) / 2;
  int64_t* conn = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t w0 = 0, assigned = 0, cur = seed;
  for (;;) {
    side[cur] = 0;
    w0 += ug->nw[cur];
    ++assigned;
    for (int64_t e = ug->off[cur]; e < ug->off[cur + 1]; ++e)
      if (side[ug->adj[e]] == 1) conn[ug->adj[e]] += ug->ew[e];
    if (w0 >= target || assigned == n) break;
    int64_t best = -1, best_c = -1;
    for (int64_t v = 0; v < n; ++v) {
      if (side[v] == 0) continue;
      if (conn[v] > best_c || (conn[v] == best_c && (best == -1 || v < best))) {
        best_c = conn[v];
        best = v;
      }
    }
    if (best == -1) break;
    cur = best;
  }
  free(conn);
}

/* exact_rebalance: partition.cpp:281-305 */
static void exact_rebalance(const ugraph* ug, int* side) {
  int64_t side_w[2] = {0, 0};
  for (int64_t v = 0; v < ug->n; ++v) side_w[side[v]] += ug->nw[v];
  while (i64abs(side_w[0] - side_w[1]) > 1) {
    int from = side_w[0] > side_w[1] ? 0 : 1;
    int64_t best = -1, best_gain = 0;
    for (int64_t v = 0; v < ug->n; ++v) {
      if (side[v] != from) continue;
      if (2 * ug->nw[v] > side_w[from] - side_w[1 - from]) continue;
      int64_t g = 0;
      for (int64_t e = ug->off[v]; e < ug->off[v + 1]; ++e)
        g += (side[ug->adj[e]] != from) ? ug->ew[e] : -ug->ew[e];
      if (best == -1 || g > best_gain || (g == best_gain && v < best)) {
        best = v;
        best_gain = g;
      }
    }
    if (best == -1) break;
    side[best] = 1 - from;
    side_w[from] -= ug->nw[best];
    side_w[1 - from] += ug->nw[best];
  }
}

/* bisect: coarsen to <= 64 nodes (stop if < 5% shrink), 4 grow+FM restarts,
 * project + FM per level, exact rebalance, FM polish. partition.cpp:310-350 */
static int* bisect(const ugraph* ug0, orc_mt64* rng) {
  int* side_out;
  if (ug0->n == 1) {
    side_out = (int*)malloc(sizeof(int));
    side_out[0] = 0;
    return side_out;
  }
  int64_t cap = 64, nlev = 1;
  ugraph* levels = (ugraph*)calloc((size_t)cap, sizeof(ugraph));
  int64_t** maps = (int64_t**)calloc((size_t)cap, sizeof(int64_t*));
  levels[0] = *ug0; /* borrowed; never freed here */
  while (levels[nlev - 1].n > 64) {
    const ugraph* cur = &levels[nlev - 1];
    int64_t* partner = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cur->n + 1));
    heavy_edge_matching(cur, rng, partner);
    ugraph coarse;
    memset(&coarse, 0, sizeof coarse);
    int64_t* f2c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cur->n + 1));
    contract(cur, partner, &coarse, f2c);
    free(partner);
    if ((double)coarse.n > 0.95 * (double)cur->n) {
      ug_free(&coarse);
      free(f2c);
      break;
    }
    if (nlev == cap) {
      cap *= 2;
      levels = (ugraph*)realloc(levels, sizeof(ugraph) * (size_t)cap);
      maps = (int64_t**)realloc(maps, sizeof(int64_t*) * (size_t)cap);
    }
    maps[nlev - 1] = f2c;
    levels[nlev++] = coarse;
  }
  const ugraph* coarsest = &levels[nlev - 1];
  int* side = NULL;
  int64_t best_cut = -1;
  int* dist = (int*)malloc(sizeof(int) * (size_t)(coarsest->n + 1));
  int* cand = NULL;
  for (int r = 0; r < 4; ++r) {
    int64_t u1 = farthest_from(coarsest, orc_uniform_int(rng, 0, coarsest->n - 1), dist);
    int64_t seed = farthest_from(coarsest, u1, dist);
    int64_t start = (r == 0) ? seed : orc_uniform_int(rng, 0, coarsest->n - 1);
    cand = (int*)malloc(sizeof(int) * (size_t)(coarsest->n + 1));
    grow_region(coarsest, start, cand);
    fm_refine(coarsest, cand, balance_allowance(coarsest));
    int64_t cut = cut_weight(coarsest, cand);
    if (best_cut < 0 || cut < best_cut) {
      best_cut = cut;
      free(side);
      side = cand;
    } else {
      free(cand);
    }
  }
  free(dist);
  for (int64_t level = nlev - 1; level-- > 0;) {
    int64_t nf = levels[level].n;
    int* fine = (int*)malloc(sizeof(int) * (size_t)(nf + 1));
    for (int64_t v = 0; v < nf; ++v) fine[v] = side[maps[level][v]];
    free(side);
    side = fine;
    fm_refine(&levels[level], side, balance_allowance(&levels[level]));
  }
  exact_rebalance(ug0, side);
  fm_refine(ug0, side, 1);
  for (int64_t l = 1; l < nlev; ++l) ug_free(&levels[l]);
  for (int64_t l = 0; l + 1 < nlev; ++l) free(maps[l]);
  free(levels);
  free(maps);
  return side;
}

/* recursive_bisect: partition.cpp:352-391 */
static void recursive_bisect(const ugraph* ug, const int64_t* ids, int64_t k, uint64_t seed,
                             int64_t part_base, int64_t* part_of) {
  if (k == 1 || ug->n == 0) {
    for (int64_t v = 0; v < ug->n; ++v) part_of[ids[v]] = part_base;
    return;
  }
  orc_mt64 rng;
  orc_mt64_seed(&rng, orc_splitmix64(seed));
  int* side = bisect(ug, &rng);
  int64_t* sub_id = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ug->n + 1));
  int64_t cnt[2] = {0, 0};
  for (int64_t v = 0; v < ug->n; ++v) sub_id[v] = cnt[side[v]]++;
  ugraph sub[2];
  int64_t* ids_sub[2];
  for (int s = 0; s < 2; ++s) {
    memset(&sub[s], 0, sizeof(ugraph));
    sub[s].n = cnt[s];
    sub[s].off = (int64_t*)calloc((size_t)cnt[s] + 1, sizeof(int64_t));
    sub[s].nw = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cnt[s] + 1));
    sub[s].adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ug->m + 1));
    sub[s].ew = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ug->m + 1));
    ids_sub[s] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cnt[s] + 1));
  }
  for (int64_t v = 0; v < ug->n; ++v) {
    int s = side[v];
    ids_sub[s][sub_id[v]] = ids[v];
    sub[s].nw[sub_id[v]] = ug->nw[v];
  }
  for (int64_t v = 0; v < ug->n; ++v) {
    int s = side[v];
    for (int64_t e = ug->off[v]; e < ug->off[v + 1]; ++e) {
      if (side[ug->adj[e]] != s) continue;
      sub[s].adj[sub[s].m] = sub_id[ug->adj[e]];
      sub[s].ew[sub[s].m] = ug->ew[e];
      sub[s].m++;
    }
    sub[s].off[sub_id[v] + 1] = sub[s].m;
  }
  for (int s = 0; s < 2; ++s)
    for (int64_t u = 0; u < sub[s].n; ++u)
      if (sub[s].off[u + 1] < sub[s].off[u]) sub[s].off[u + 1] = sub[s].off[u];
  free(side);
  free(sub_id);
  recursive_bisect(&sub[0], ids_sub[0], k / 2, orc_splitmix64(seed ^ 0x517cc1b727220a95ULL),
                   part_base, part_of);
  recursive_bisect(&sub[1], ids_sub[1], k / 2, orc_splitmix64(seed ^ 0x2545f4914f6cdd1dULL),
                   part_base + k / 2, part_of);
  for (int s = 0; s < 2; ++s) {
    ug_free(&sub[s]);
    free(ids_sub[s]);
  }
}

/* reorder: partition.cpp:413-433 (stable sort by part id == counting sort). */
int orc_reorder(const orc_csr* g, int64_t k, uint64_t seed, int64_t* forward, int64_t* inverse) {
  if (k < 1 || (k & (k - 1)) != 0) return orc_fail(ORC_CONFIG, "reorder: k must be a power of two >= 1");
  if (k > g->n) return orc_fail(ORC_CONFIG, "reorder: k exceeds node count");
  ugraph ug;
  memset(&ug, 0, sizeof ug);
  ugraph_from(g, &ug);
  int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n + 1));
  for (int64_t i = 0; i < g->n; ++i) ids[i] = i;
  int64_t* part = (int64_t*)calloc((size_t)g->n + 1, sizeof(int64_t));
  recursive_bisect(&ug, ids, k, orc_splitmix64(seed ^ 0xda3e39cb94b95bdbULL), 0, part);
  int64_t pos = 0;
  for (int64_t p = 0; p < k; ++p)
    for (int64_t v = 0; v < g->n; ++v)
      if (part[v] == p) inverse[pos++] = v;
  for (int64_t q = 0; q < g->n; ++q) forward[inverse[q]] = q;
  free(ids);
  free(part);
  ug_free(&ug);
  return ORC_OK;
}

static int perm_valid(int64_t n, const int64_t* fwd) {
  char* seen = (char*)calloc((size_t)n + 1, 1);
  int ok = 1;
  for (int64_t i = 0; i < n && ok; ++i) {
    if (fwd[i] < 0 || fwd[i] >= n || seen[fwd[i]]) ok = 0;
    else seen[fwd[i]] = 1;
  }
  free(seen);
  return ok;
}

/* permute_graph: relabel then graph_from_edges. partition.cpp:435-456 */
int orc_permute_graph(const orc_csr* g, const int64_t* forward, orc_csr* out) {
  if (!perm_valid(g->n, forward)) return orc_fail(ORC_CONFIG, "permute_graph: bad permutation");
  int64_t* s = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->nnz + 1));
  int64_t* d = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->nnz + 1));
  for (int64_t u = 0; u < g->n; ++u)
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      s[e] = forward[u];
      d[e] = forward[g->cols[e]];
    }
  int rc = orc_graph_from_edges(g->n, g->nnz, s, d, out);
  free(s);
  free(d);
  return rc;
}

/* cluster_boundaries: partition.cpp:495-500 */
void orc_cluster_boundaries(int64_t n, int64_t k, int64_t* b) {
  int64_t base = n / k, rem = n % k;
  b[0] = 0;
  for (int64_t i = 0; i < k; ++i) b[i + 1] = b[i] + base + (i < rem ? 1 : 0);
}

/* ClusterGrid::cluster_of: partition.cpp:502-508 */
int64_t orc_cluster_of(int64_t n, int64_t k, int64_t pos) {
  int64_t base = n / k, rem = n % k, cut = rem * (base + 1);
  if (pos < cut) return pos / (base + 1);
  return rem + (pos - cut) / base;
}

/* build_cluster_grid: partition.cpp:514-539 */
int orc_build_cluster_grid(const orc_csr* g, const int64_t* forward, int64_t k, int64_t* bnd,
                           int64_t* cell_nnz, double* cell_density) {
  if (k < 1 || k > g->n) return orc_fail(ORC_CONFIG, "build_cluster_grid: invalid k");
  if (!perm_valid(g->n, forward))
    return orc_fail(ORC_CONFIG, "build_cluster_grid: permutation does not match graph");
  orc_cluster_boundaries(g->n, k, bnd);
  for (int64_t c = 0; c < k * k; ++c) cell_nnz[c] = 0;
  for (int64_t u = 0; u < g->n; ++u) {
    int64_t a = orc_cluster_of(g->n, k, forward[u]);
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e)
      cell_nnz[a * k + orc_cluster_of(g->n, k, forward[g->cols[e]])]++;
  }
  for (int64_t a = 0; a < k; ++a)
    for (int64_t b = 0; b < k; ++b) {
      double area = (double)(bnd[a + 1] - bnd[a]) * (double)(bnd[b + 1] - bnd[b]);
      cell_density[a * k + b] = (double)cell_nnz[a * k + b] / area;
    }
  return ORC_OK;
}

/* diagonal_edge_fraction: partition.cpp:541-547 */
int orc_diagonal_edge_fraction(int64_t k, const int64_t* cell_nnz, double* out) {
  int64_t total = 0, diag = 0;
  for (int64_t c = 0; c < k * k; ++c) total += cell_nnz[c];
  if (total == 0) return orc_fail(ORC_DATA, "diagonal_edge_fraction: empty graph");
  for (int64_t a = 0; a < k; ++a) diag += cell_nnz[a * k + a];
  *out = (double)diag / (double)total;
  return ORC_OK;
}

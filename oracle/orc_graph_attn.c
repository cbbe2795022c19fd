/* TEST INFRASTRUCTURE — not product code. CPU oracle, see oracle.h.
 * Graph CSR builders and fp64 attention, restated from
 *   /root/reference/proj/src/graph.cpp and /root/reference/proj/src/attention.cpp.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

int orc_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void orc_csr_free(orc_csr* g) {
  if (!g) return;
  free(g->row_off);
  free(g->cols);
  g->row_off = g->cols = NULL;
  g->n = g->nnz = 0;
}

typedef struct {
  int64_t u, v;
} pair64;

static int cmp_pair(const void* a, const void* b) {
  const pair64* x = (const pair64*)a;
  const pair64* y = (const pair64*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}

/* graph_from_edges: range check, sort + unique, counting offsets.
 * Reference: proj/src/graph.cpp:49-66 (range check :18-23). */
int orc_graph_from_edges(int64_t n, int64_t m, const int64_t* src, const int64_t* dst, orc_csr* out) {
  if (n < 0) return orc_fail(ORC_DATA, "graph_from_edges: negative node count");
  for (int64_t e = 0; e < m; ++e) {
    const int64_t ends[2] = {src[e], dst[e]};
    for (int t = 0; t < 2; ++t) {
      if (ends[t] < 0 || ends[t] >= n) {
        return orc_fail(ORC_DATA, "graph_from_edges: node id %lld out of range [0, %lld)",
                        (long long)ends[t], (long long)n);
      }
    }
  }
  pair64* p = (pair64*)malloc(sizeof(pair64) * (size_t)(m > 0 ? m : 1));
  for (int64_t e = 0; e < m; ++e) {
    p[e].u = src[e];
    p[e].v = dst[e];
  }
  qsort(p, (size_t)m, sizeof(pair64), cmp_pair);
  int64_t w = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (w == 0 || p[e].u != p[w - 1].u || p[e].v != p[w - 1].v) p[w++] = p[e];
  }
  out->n = n;
  out->nnz = w;
  out->row_off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  out->cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(w > 0 ? w : 1));
  for (int64_t e = 0; e < w; ++e) out->row_off[p[e].u + 1]++;
  for (int64_t i = 0; i < n; ++i) out->row_off[i + 1] += out->row_off[i];
  for (int64_t e = 0; e < w; ++e) out->cols[e] = p[e].v;
  free(p);
  return ORC_OK;
}

/* add_self_loops: insert (u,u) at its sorted slot when absent; idempotent.
 * Reference: proj/src/graph.cpp:127-149. */
int orc_add_self_loops(const orc_csr* g, orc_csr* out) {
  out->n = g->n;
  out->row_off = (int64_t*)calloc((size_t)g->n + 1, sizeof(int64_t));
  out->cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->nnz + g->n + 1));
  int64_t w = 0;
  for (int64_t u = 0; u < g->n; ++u) {
    int placed = 0;
    for (int64_t e = g->row_off[u]; e < g->row_off[u + 1]; ++e) {
      int64_t v = g->cols[e];
      if (!placed && v >= u) {
        if (v != u) out->cols[w++] = u;
        placed = 1;
      }
      out->cols[w++] = v;
    }
    if (!placed) out->cols[w++] = u;
    out->row_off[u + 1] = w;
  }
  out->nnz = w;
  return ORC_OK;
}

/* density = nnz / (N*N) in double. Reference: proj/src/graph.cpp:151-155. */
int orc_density(const orc_csr* g, double* out) {
  if (g->n < 1) return orc_fail(ORC_DATA, "density: empty graph");
  *out = (double)g->nnz / ((double)g->n * (double)g->n);
  return ORC_OK;
}

static int all_finite(const double* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

static int check_finite3(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                         const double* v) {
  /* proj/src/attention.cpp:20-22 — checked in Q, K, V order */
  if (!all_finite(q, S * dk)) return orc_fail(ORC_DATA, "attention: non-finite Q");
  if (!all_finite(k, S * dk)) return orc_fail(ORC_DATA, "attention: non-finite K");
  if (!all_finite(v, S * dv)) return orc_fail(ORC_DATA, "attention: non-finite V");
  return ORC_OK;
}

/* sparse_attention: per row SDDMM -> max -> exp -> normalise -> SpMM.
 * Reference: proj/src/attention.cpp:96-162 (deg 0 :119-125, deg 1 :128-135,
 * general :136-157). */
int orc_sparse_attn_fwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                        const double* v, const int64_t* row_off, const int64_t* cols,
                        const double* bias, const double* wmult, int forbid_empty, double* out) {
  if (dk < 1) return orc_fail(ORC_CONFIG, "attention: d_K must be >= 1");
  int rc = check_finite3(S, dk, dv, q, k, v);
  if (rc) return rc;
  const double scale = 1.0 / sqrt((double)dk);
  memset(out, 0, sizeof(double) * (size_t)(S * dv));
  int64_t maxdeg = 1;
  for (int64_t i = 0; i < S; ++i) {
    int64_t d = row_off[i + 1] - row_off[i];
    if (d > maxdeg) maxdeg = d;
  }
  double* sc = (double*)malloc(sizeof(double) * (size_t)maxdeg);
  for (int64_t i = 0; i < S; ++i) {
    const int64_t b = row_off[i], e1 = row_off[i + 1], deg = e1 - b;
    if (deg == 0) {
      if (forbid_empty) {
        free(sc);
        return orc_fail(ORC_DATA, "sparse_attention: row %lld attends to nothing; run add_self_loops",
                        (long long)i);
      }
      continue;
    }
    double* o = out + i * dv;
    const double* qi = q + i * dk;
    if (deg == 1) {
      double w = wmult ? wmult[b] : 1.0;
      const double* vj = v + cols[b] * dv;
      for (int64_t t = 0; t < dv; ++t) o[t] = w * vj[t];
      continue;
    }
    double mx = -INFINITY;
    for (int64_t e = b; e < e1; ++e) {
      const double* kj = k + cols[e] * dk;
      double acc = 0;
      for (int64_t t = 0; t < dk; ++t) acc += qi[t] * kj[t];
      acc *= scale;
      if (bias) acc += bias[e];
      sc[e - b] = acc;
      if (acc > mx) mx = acc;
    }
    double denom = 0;
    for (int64_t e = 0; e < deg; ++e) {
      sc[e] = exp(sc[e] - mx);
      denom += sc[e];
    }
    for (int64_t e = b; e < e1; ++e) {
      double w = sc[e - b] / denom;
      if (wmult) w *= wmult[e];
      const double* vj = v + cols[e] * dv;
      for (int64_t t = 0; t < dv; ++t) o[t] += w * vj[t];
    }
  }
  free(sc);
  return ORC_OK;
}

/* sparse_attention_backward: recompute softmax, dV scatter, dw/dot, ds, dQ/dK.
 * Reference: proj/src/attention.cpp:241-320 (deg 1 :265-272). No finiteness
 * check, as in the reference. */
int orc_sparse_attn_bwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                        const double* v, const int64_t* row_off, const int64_t* cols,
                        const double* bias, const double* wmult, const double* up, double* dq,
                        double* dkk, double* dvv, double* dbias) {
  if (dk < 1) return orc_fail(ORC_CONFIG, "attention: d_K must be >= 1");
  const double scale = 1.0 / sqrt((double)dk);
  memset(dq, 0, sizeof(double) * (size_t)(S * dk));
  memset(dkk, 0, sizeof(double) * (size_t)(S * dk));
  memset(dvv, 0, sizeof(double) * (size_t)(S * dv));
  memset(dbias, 0, sizeof(double) * (size_t)row_off[S]);
  int64_t maxdeg = 1;
  for (int64_t i = 0; i < S; ++i) {
    int64_t d = row_off[i + 1] - row_off[i];
    if (d > maxdeg) maxdeg = d;
  }
  double* w = (double*)malloc(sizeof(double) * (size_t)maxdeg);
  double* dw = (double*)malloc(sizeof(double) * (size_t)maxdeg);
  for (int64_t i = 0; i < S; ++i) {
    const int64_t b = row_off[i], e1 = row_off[i + 1], deg = e1 - b;
    if (deg == 0) continue;
    const double* qi = q + i * dk;
    const double* ui = up + i * dv;
    if (deg == 1) {
      int64_t j = cols[b];
      double m = wmult ? wmult[b] : 1.0;
      double* dvj = dvv + j * dv;
      for (int64_t t = 0; t < dv; ++t) dvj[t] += m * ui[t];
      continue;
    }
    double mx = -INFINITY;
    for (int64_t e = b; e < e1; ++e) {
      const double* kj = k + cols[e] * dk;
      double acc = 0;
      for (int64_t t = 0; t < dk; ++t) acc += qi[t] * kj[t];
      acc *= scale;
      if (bias) acc += bias[e];
      w[e - b] = acc;
      if (acc > mx) mx = acc;
    }
    double denom = 0;
    for (int64_t e = 0; e < deg; ++e) {
      w[e] = exp(w[e] - mx);
      denom += w[e];
    }
    for (int64_t e = 0; e < deg; ++e) w[e] /= denom;
    double dot = 0;
    for (int64_t e = b; e < e1; ++e) {
      int64_t j = cols[e];
      double m = wmult ? wmult[e] : 1.0;
      const double* vj = v + j * dv;
      double dwj = 0;
      for (int64_t t = 0; t < dv; ++t) dwj += ui[t] * vj[t];
      double* dvj = dvv + j * dv;
      double wm = w[e - b] * m;
      for (int64_t t = 0; t < dv; ++t) dvj[t] += wm * ui[t];
      dw[e - b] = dwj * m;
      dot += w[e - b] * dw[e - b];
    }
    double* dqi = dq + i * dk;
    for (int64_t e = b; e < e1; ++e) {
      int64_t j = cols[e];
      double ds = w[e - b] * (dw[e - b] - dot);
      dbias[e] = ds;
      const double* kj = k + j * dk;
      double* dkj = dkk + j * dk;
      double dss = ds * scale;
      for (int64_t t = 0; t < dk; ++t) {
        dqi[t] += dss * kj[t];
        dkj[t] += dss * qi[t];
      }
    }
  }
  free(w);
  free(dw);
  return ORC_OK;
}

/* dense_attention: reference proj/src/attention.cpp:46-94. */
int orc_dense_attn_fwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                       const double* v, const double* bias, const double* wmult, double* out) {
  if (dk < 1) return orc_fail(ORC_CONFIG, "attention: d_K must be >= 1");
  int rc = check_finite3(S, dk, dv, q, k, v);
  if (rc) return rc;
  if (bias && !all_finite(bias, S * S)) return orc_fail(ORC_DATA, "attention: non-finite bias");
  const double scale = 1.0 / sqrt((double)dk);
  memset(out, 0, sizeof(double) * (size_t)(S * dv));
  double* sc = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
  for (int64_t i = 0; i < S; ++i) {
    const double* qi = q + i * dk;
    double mx = -INFINITY;
    for (int64_t j = 0; j < S; ++j) {
      const double* kj = k + j * dk;
      double acc = 0;
      for (int64_t t = 0; t < dk; ++t) acc += qi[t] * kj[t];
      acc *= scale;
      if (bias) acc += bias[i * S + j];
      sc[j] = acc;
      if (acc > mx) mx = acc;
    }
    double denom = 0;
    for (int64_t j = 0; j < S; ++j) {
      sc[j] = exp(sc[j] - mx);
      denom += sc[j];
    }
    double* o = out + i * dv;
    for (int64_t j = 0; j < S; ++j) {
      double w = sc[j] / denom;
      if (wmult) w *= wmult[i * S + j];
      const double* vj = v + j * dv;
      for (int64_t t = 0; t < dv; ++t) o[t] += w * vj[t];
    }
  }
  free(sc);
  return ORC_OK;
}

/* dense_attention_backward: reference proj/src/attention.cpp:174-239. */
int orc_dense_attn_bwd(int64_t S, int64_t dk, int64_t dv, const double* q, const double* k,
                       const double* v, const double* bias, const double* wmult,
                       const double* up, double* dq, double* dkk, double* dvv, double* dbias) {
  if (dk < 1) return orc_fail(ORC_CONFIG, "attention: d_K must be >= 1");
  const double scale = 1.0 / sqrt((double)dk);
  memset(dq, 0, sizeof(double) * (size_t)(S * dk));
  memset(dkk, 0, sizeof(double) * (size_t)(S * dk));
  memset(dvv, 0, sizeof(double) * (size_t)(S * dv));
  memset(dbias, 0, sizeof(double) * (size_t)(S * S));
  double* w = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
  double* dw = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
  for (int64_t i = 0; i < S; ++i) {
    const double* qi = q + i * dk;
    double mx = -INFINITY;
    for (int64_t j = 0; j < S; ++j) {
      const double* kj = k + j * dk;
      double acc = 0;
      for (int64_t t = 0; t < dk; ++t) acc += qi[t] * kj[t];
      acc *= scale;
      if (bias) acc += bias[i * S + j];
      w[j] = acc;
      if (acc > mx) mx = acc;
    }
    double denom = 0;
    for (int64_t j = 0; j < S; ++j) {
      w[j] = exp(w[j] - mx);
      denom += w[j];
    }
    for (int64_t j = 0; j < S; ++j) w[j] /= denom;
    const double* ui = up + i * dv;
    double dot = 0;
    for (int64_t j = 0; j < S; ++j) {
      const double* vj = v + j * dv;
      double m = wmult ? wmult[i * S + j] : 1.0;
      double dwj = 0;
      for (int64_t t = 0; t < dv; ++t) dwj += ui[t] * vj[t];
      double* dvj = dvv + j * dv;
      double wm = w[j] * m;
      for (int64_t t = 0; t < dv; ++t) dvj[t] += wm * ui[t];
      dw[j] = dwj * m;
      dot += w[j] * dw[j];
    }
    double* dqi = dq + i * dk;
    for (int64_t j = 0; j < S; ++j) {
      double ds = w[j] * (dw[j] - dot);
      dbias[i * S + j] = ds;
      const double* kj = k + j * dk;
      double* dkj = dkk + j * dk;
      double dss = ds * scale;
      for (int64_t t = 0; t < dk; ++t) {
        dqi[t] += dss * kj[t];
        dkj[t] += dss * qi[t];
      }
    }
  }
  free(w);
  free(dw);
  return ORC_OK;
}

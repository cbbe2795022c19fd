/* TEST INFRASTRUCTURE — not product code. CPU oracle, see oracle.h.
 * Sequence-parallel layer restated serially from
 *   /root/reference/proj/src/parallel.cpp:83-332.
 * Workers are logical: the all-to-alls are index arithmetic plus the element
 * ledger, exactly as in the reference.
 */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "orc_rng.h"

int orc_fail(int code, const char* fmt, ...);

/* partition_sequence: pad to a multiple of P, shuffle ids, split
 * contiguously. parallel.cpp:96-113 */
int orc_partition_sequence(int64_t S, int64_t P, uint64_t seed, int64_t* ids, int64_t* padded) {
  if (P < 1) return orc_fail(ORC_CONFIG, "partition_sequence: worker count must be >= 1");
  if (S < 1) return orc_fail(ORC_CONFIG, "partition_sequence: empty sequence");
  const int64_t pad = ((S + P - 1) / P) * P;
  for (int64_t i = 0; i < pad; ++i) ids[i] = i;
  orc_mt64 rng;
  orc_mt64_seed(&rng, seed);
  orc_shuffle_i64(ids, pad, &rng);
  *padded = pad;
  return ORC_OK;
}

static int check_div(int64_t d, int64_t H, int64_t P) {
  if (H % P != 0) return orc_fail(ORC_CONFIG, "all_to_all: head count not divisible by worker count");
  if (d % H != 0) return orc_fail(ORC_CONFIG, "all_to_all: hidden dim not divisible by head count");
  return ORC_OK;
}

/* Per worker w, the full token-indexed slice [S_pad x d/P] it holds after
 * all_to_all_seq_to_head (parallel.cpp:115-147): out_w[token] = x[token][w*sl : (w+1)*sl].
 * Ledger: each source worker sends rows*slice to each destination. */
static void gather_slice(int64_t S_pad, int64_t d, int64_t P, int64_t w, const double* x, double* out) {
  const int64_t sl = d / P;
  for (int64_t t = 0; t < S_pad; ++t) memcpy(out + t * sl, x + t * d + w * sl, sizeof(double) * (size_t)sl);
}

/* run_distributed_layer (pattern form): parallel.cpp:190-252.
 * ledger columns: qkv_gather, qkv_gather_cross, output_scatter,
 * output_scatter_cross, bias_exchange. */
int orc_dist_layer_fwd(int64_t P, int64_t S_pad, int64_t d, int64_t H, const int64_t* ids,
                       const double* q, const double* k, const double* v,
                       const int64_t* row_off, const int64_t* cols, const int64_t* perm_fwd,
                       const int64_t* perm_inv, const double* bias, int64_t nbias,
                       const double* wmult, double* out, int64_t* ledger, int64_t* score_macs) {
  (void)ids;
  int rc = check_div(d, H, P);
  if (rc) return rc;
  const int64_t hd = d / H, hpw = H / P, sl = d / P, rows = S_pad / P, nnz = row_off[S_pad];
  memset(ledger, 0, sizeof(int64_t) * (size_t)(5 * P));
  /* three seq->head exchanges (Q, K, V), counted as qkv */
  for (int rep = 0; rep < 3; ++rep)
    for (int64_t src = 0; src < P; ++src)
      for (int64_t dst = 0; dst < P; ++dst) {
        ledger[src * 5 + 0] += rows * sl;
        if (dst != src) ledger[src * 5 + 1] += rows * sl;
      }
  if (nbias > 0)
    for (int64_t w = 0; w < P; ++w) ledger[w * 5 + 4] += nbias;
  double* qs = (double*)malloc(sizeof(double) * (size_t)(S_pad * sl));
  double* ks = (double*)malloc(sizeof(double) * (size_t)(S_pad * sl));
  double* vs = (double*)malloc(sizeof(double) * (size_t)(S_pad * sl));
  double* qh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* kh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* vh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* oh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  *score_macs = 0;
  for (int64_t w = 0; w < P && rc == ORC_OK; ++w) {
    gather_slice(S_pad, d, P, w, q, qs);
    gather_slice(S_pad, d, P, w, k, ks);
    gather_slice(S_pad, d, P, w, v, vs);
    for (int64_t t = 0; t < hpw && rc == ORC_OK; ++t) {
      const int64_t h = w * hpw + t;
      /* permute_rows (row r <- token perm_inv[r]) then slice_cols: parallel.cpp:48-73 */
      for (int64_t r = 0; r < S_pad; ++r) {
        memcpy(qh + r * hd, qs + perm_inv[r] * sl + t * hd, sizeof(double) * (size_t)hd);
        memcpy(kh + r * hd, ks + perm_inv[r] * sl + t * hd, sizeof(double) * (size_t)hd);
        memcpy(vh + r * hd, vs + perm_inv[r] * sl + t * hd, sizeof(double) * (size_t)hd);
      }
      rc = orc_sparse_attn_fwd(S_pad, hd, hd, qh, kh, vh, row_off, cols, bias,
                               wmult ? wmult + h * nnz : NULL, 0, oh);
      *score_macs += nnz * hd;
      /* unpermute_rows (token t <- row perm_fwd[t]) + place_cols + scatter */
      for (int64_t tok = 0; tok < S_pad; ++tok)
        memcpy(out + tok * d + h * hd, oh + perm_fwd[tok] * hd, sizeof(double) * (size_t)hd);
    }
  }
  /* head->seq exchange of O, counted as output_scatter: parallel.cpp:149-188 */
  for (int64_t src = 0; src < P; ++src)
    for (int64_t dst = 0; dst < P; ++dst) {
      ledger[src * 5 + 2] += rows * sl;
      if (dst != src) ledger[src * 5 + 3] += rows * sl;
    }
  free(qs); free(ks); free(vs); free(qh); free(kh); free(vh); free(oh);
  return rc;
}

/* run_distributed_layer_backward: parallel.cpp:271-332; dbias summed over
 * heads in worker-then-head order (:319). */
int orc_dist_layer_bwd(int64_t P, int64_t S_pad, int64_t d, int64_t H, const int64_t* ids,
                       const double* q, const double* k, const double* v,
                       const int64_t* row_off, const int64_t* cols, const int64_t* perm_fwd,
                       const int64_t* perm_inv, const double* bias, const double* wmult,
                       const double* up, double* dq, double* dkk, double* dvv, double* dbias) {
  (void)ids;
  int rc = check_div(d, H, P);
  if (rc) return rc;
  const int64_t hd = d / H, hpw = H / P, nnz = row_off[S_pad];
  memset(dbias, 0, sizeof(double) * (size_t)nnz);
  double* qh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* kh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* vh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* uh = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* gq = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* gk = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* gv = (double*)malloc(sizeof(double) * (size_t)(S_pad * hd));
  double* gb = (double*)malloc(sizeof(double) * (size_t)(nnz + 1));
  for (int64_t w = 0; w < P && rc == ORC_OK; ++w) {
    for (int64_t t = 0; t < hpw && rc == ORC_OK; ++t) {
      const int64_t h = w * hpw + t;
      for (int64_t r = 0; r < S_pad; ++r) {
        int64_t tok = perm_inv[r];
        memcpy(qh + r * hd, q + tok * d + h * hd, sizeof(double) * (size_t)hd);
        memcpy(kh + r * hd, k + tok * d + h * hd, sizeof(double) * (size_t)hd);
        memcpy(vh + r * hd, v + tok * d + h * hd, sizeof(double) * (size_t)hd);
        memcpy(uh + r * hd, up + tok * d + h * hd, sizeof(double) * (size_t)hd);
      }
      rc = orc_sparse_attn_bwd(S_pad, hd, hd, qh, kh, vh, row_off, cols, bias,
                               wmult ? wmult + h * nnz : NULL, uh, gq, gk, gv, gb);
      for (int64_t p = 0; p < nnz; ++p) dbias[p] += gb[p];
      for (int64_t tok = 0; tok < S_pad; ++tok) {
        int64_t r = perm_fwd[tok];
        memcpy(dq + tok * d + h * hd, gq + r * hd, sizeof(double) * (size_t)hd);
        memcpy(dkk + tok * d + h * hd, gk + r * hd, sizeof(double) * (size_t)hd);
        memcpy(dvv + tok * d + h * hd, gv + r * hd, sizeof(double) * (size_t)hd);
      }
    }
  }
  free(qh); free(kh); free(vh); free(uh); free(gq); free(gk); free(gv); free(gb);
  return rc;
}

/* ---- Trainer glue ---- */

/* proj/src/model.cpp:76-83 */
int orc_extend_with_pad_loops(const orc_csr* pat, int64_t s_pad, orc_csr* out) {
  const int64_t n = pat->n, extra = s_pad > n ? s_pad - n : 0;
  out->n = n + extra;
  out->nnz = pat->nnz + extra;
  out->row_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(out->n + 1));
  out->cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(out->nnz > 0 ? out->nnz : 1));
  for (int64_t r = 0; r <= n; ++r) out->row_off[r] = pat->row_off[r];
  for (int64_t e = 0; e < pat->nnz; ++e) out->cols[e] = pat->cols[e];
  for (int64_t r = n; r < n + extra; ++r) {
    out->cols[out->row_off[r]] = r;
    out->row_off[r + 1] = out->row_off[r] + 1;
  }
  return ORC_OK;
}

/* SpdTable::lookup, proj/src/graph.cpp:208-214 (lower_bound in row i) */
static int64_t spd_lookup(const int64_t* ro, const int64_t* cols, const uint16_t* dist, int64_t i, int64_t j,
                          int64_t unreachable) {
  int64_t lo = ro[i], hi = ro[i + 1];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (cols[mid] < j) lo = mid + 1; else hi = mid;
  }
  if (lo < ro[i + 1] && cols[lo] == j) return dist[lo];
  return unreachable;
}

/* proj/src/model.cpp:447-463 (layout_for) / :407-423 (bucket_of) */
int orc_pattern_buckets(const orc_csr* pat, const int64_t* perm_inv, int64_t global_index, int64_t spd_n,
                        const int64_t* spd_row_off, const int64_t* spd_cols, const uint16_t* spd_dist,
                        int64_t max_dist, int32_t* buckets) {
  int64_t p = 0;
  for (int64_t r = 0; r < pat->n; ++r) {
    for (int64_t e = pat->row_off[r]; e < pat->row_off[r + 1]; ++e) {
      const int64_t i = perm_inv[r], j = perm_inv[pat->cols[e]];
      int64_t b;
      if (i == j) b = 0;
      else if (i == global_index || j == global_index) b = 1;
      else if (i >= spd_n || j >= spd_n) b = max_dist + 1;
      else b = spd_lookup(spd_row_off, spd_cols, spd_dist, i, j, max_dist + 1);
      buckets[p++] = (int32_t)b;
    }
  }
  return ORC_OK;
}

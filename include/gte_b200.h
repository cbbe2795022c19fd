/* gte_b200 — C ABI of the B200-native TorchGT graph-attention hot path.
 *
 * Plain pointers and sizes, no C++ or torch types. Every entry returns a
 * gte_status; on failure gte_last_error() holds a message whose wording
 * follows the reference exception it replaces, so the C++ drop-in layer
 * (integration/gte_b200_bridge.cpp, compiled against the reference's own
 * proj/include/gte headers) can rethrow ConfigError/DataError with the same
 * substrings (reference error taxonomy: proj/include/gte/types.hpp:13-24).
 *
 * Device-pointer entries are stream-ordered on the context's stream and do not
 * synchronise; data-dependent errors (non-finite Q/K/V, empty rows under
 * GTE_FORBID_EMPTY_ROWS) are latched on the device and reported by the next
 * gte_ctx_sync() (or by any *_host entry, which synchronises).
 *
 * Index limits on the device: nnz < 2^31 and rows < 2^31 (int32 CSR/CSC).
 */
#ifndef GTE_B200_H
#define GTE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GTE_OK = 0,
  GTE_CONFIG = 2,     /* gte::ConfigError  (CLI exit 2) */
  GTE_DATA = 3,       /* gte::DataError    (CLI exit 3) */
  GTE_DIVERGENCE = 4, /* gte::DivergenceError          */
  GTE_CUDA = 5,
  GTE_NCCL = 6
} gte_status;

typedef enum { GTE_F64 = 0, GTE_F32 = 1, GTE_BF16 = 2 } gte_dtype;

/* flags: GTE_FORBID_EMPTY_ROWS raises DataError on a row with no pairs
 * (edge_sparse_attention, attention.cpp:119-123); GTE_IGNORE_NONFINITE skips
 * the Q/K/V finiteness error (the reference's backward recomputes the softmax
 * without checking, attention.cpp:241-320). */
enum { GTE_FORBID_EMPTY_ROWS = 1, GTE_IGNORE_NONFINITE = 2 };

typedef struct gte_ctx gte_ctx;
typedef struct gte_plan gte_plan;

const char* gte_last_error(void);
const char* gte_version(void);

/* ---- context: device, stream, workspaces, latched device errors ---- */
int gte_ctx_create(int device, gte_ctx** out);
int gte_ctx_destroy(gte_ctx* ctx);
/* device memory for callers without the CUDA runtime (the C++ drop-in):
 * stream-ordered on the context; gte_copy_d2h synchronises */
int gte_dev_alloc(gte_ctx* ctx, int64_t bytes, void** out);
int gte_dev_free(gte_ctx* ctx, void* p);
int gte_copy_h2d(gte_ctx* ctx, void* dst, const void* src, int64_t bytes);
int gte_copy_d2h(gte_ctx* ctx, void* dst, const void* src, int64_t bytes);
int gte_ctx_set_stream(gte_ctx* ctx, void* cuda_stream);
int gte_ctx_sync(gte_ctx* ctx);
/* number of kernels this context launched so far (bench evidence) */
int64_t gte_ctx_launches(const gte_ctx* ctx);

/* ---- attention pattern plan ----
 * Replaces AttnPattern (reference proj/include/gte/attention.hpp:13-23) on the
 * device: int32 CSR + the CSC view (col_ptr, csc_row, csc_eid) the atomic-free
 * backward needs, plus the list of never-referenced rows for the finite check.
 * _host takes the reference's int64 CSR in host memory; _device takes int32
 * CSR already resident in HBM (no host round trip). */
int gte_plan_create_host(gte_ctx* ctx, int64_t rows, int64_t nnz, const int64_t* row_off,
                         const int64_t* cols, gte_plan** out);
int gte_plan_create_device(gte_ctx* ctx, int64_t rows, int64_t nnz, const int32_t* d_row_ptr,
                           const int32_t* d_cols, gte_plan** out);
int gte_plan_destroy(gte_plan* plan);
int gte_plan_shape(const gte_plan* plan, int64_t* rows, int64_t* nnz, int64_t* max_row_deg,
                   int64_t* max_col_deg);
/* device pointers of the plan's int32 CSR/CSC (for fused callers) */
int gte_plan_device_csr(const gte_plan* plan, const int32_t** row_ptr, const int32_t** cols);

/* ---- execution schedule (no reference counterpart: an execution order only;
 * results are bit-identical with or without it) ----
 * gte_community_order: host, synchronous label propagation over the
 *   symmetrised pattern (`iters` rounds max), rows ordered by (label, row);
 *   order[n] receives the row sequence (csrc/schedule.cpp).
 * gte_plan_schedule: the same on a plan's CSR, stored on the device; the
 *   sparse kernels then execute rows (and CSC columns) in that order so a
 *   CTA's gathers hit rows its neighbours just pulled into L1.
 * gte_plan_set_order: any permutation of [0, rows) (NULL clears). */
int gte_community_order(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t iters,
                        int64_t* order, int64_t* n_communities);
int gte_plan_schedule(gte_plan* plan, int64_t iters, int64_t* n_communities);
int gte_plan_set_order(gte_plan* plan, const int64_t* order);
/* Rows [n, rows) produce no outputs (forward O / LSE, dQ, the backward's
 * CSR pass skip them; the CSC pass still covers every column); they must have
 * no edges. For a sequence-parallel rank's local plan, whose halo rows exist
 * only as columns (no reference counterpart: an execution-plan option). */
int gte_plan_set_output_rows(gte_plan* plan, int64_t n);

/* ---- Elastic Computation Reformation on the tensor pipe (the
 * reference's dense sub-blocks, reformation.cpp:111-195, tile spans
 * :176-189, executed by cluster_sparse_attention :197-204) ----
 * gte_plan_set_blocks: registers the layout's d_b x d_b sub-blocks as global
 *   origins [n_blocks][2] = (row0, col0). With d_b == 16 and a bf16 call whose
 *   head geometry has tile kernels (dh in {8, 16}, H * dh in {64, 128}), their
 *   pairs run as dense 16 x 16 tiles on mma.sync and the rest of the pattern
 *   on the sparse kernels; the two merge as online-softmax partials (forward)
 *   and fixed-order partial sums (backward). Every sub-block must lie in the
 *   plan's pattern and none may overlap (ConfigError otherwise). Sub-blocks
 *   touching a row/column of degree > 1024 stay on the sparse path; other
 *   d_b register nothing. n_used: sub-blocks executed as tiles.
 * gte_plan_blocks: registered sub-blocks and the remainder's nnz. */
int gte_plan_set_blocks(gte_plan* plan, int64_t n_blocks, const int64_t* origins, int64_t d_b, int64_t* n_used);
int gte_plan_blocks(const gte_plan* plan, int64_t* n_blocks, int64_t* remainder_nnz);

/* ---- sparse (topology-induced) attention over a plan, all heads at once ----
 * Replaces sparse_attention / sparse_attention_backward (reference
 * proj/src/attention.cpp:96-162, 241-320) called per head, and the per-head
 * loop + dbias head-sum of run_distributed_layer(_backward)
 * (proj/src/parallel.cpp:234-247, 307-323).
 *
 * q, k: [S x ldq] of dtype; head h = columns [h*dk, (h+1)*dk).
 * v, out, dout: [S x ldv]; head h = columns [h*dv, (h+1)*dv).
 * bias: [nnz] (double for GTE_F64, float otherwise) shared by heads, or NULL.
 * wmult: [H x nnz] head-major post-softmax multipliers (dropout), or NULL.
 * lse: [S x H] workspace written by fwd and read by bwd (accumulate type;
 *      log2 units for f32/bf16, natural for f64).
 * dbias: [nnz] accumulate type, summed over heads (head order may differ from
 *        the reference's sequential sum by rounding only).
 * Limits: 1 <= dk, dv <= 64; H >= 1 (H > 32 processed in groups of 32). */
int gte_sparse_attn_fwd(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk, int dv,
                        const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                        const void* bias, const void* wmult, void* out, void* lse, int flags);
int gte_sparse_attn_bwd(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk, int dv,
                        const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                        const void* out, const void* lse, const void* dout, const void* bias,
                        const void* wmult, void* dq, void* dk_out, void* dv_out, void* dbias);

/* Host-pointer twins: inputs/outputs in host memory (pinned or pageable),
 * H2D/D2H copies on the context stream, synchronous; raise latched errors. */
int gte_sparse_attn_fwd_host(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk, int dv,
                             const void* q, const void* k, const void* v, const void* bias,
                             const void* wmult, void* out, void* lse_out, int flags);
int gte_sparse_attn_bwd_host(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk, int dv,
                             const void* q, const void* k, const void* v, const void* out,
                             const void* lse, const void* dout, const void* bias,
                             const void* wmult, void* dq, void* dk_out, void* dv_out,
                             void* dbias);
/* One attention sublayer, fwd + bwd, host buffers in and out (the e2e unit). */
int gte_sparse_attn_fwd_bwd_host(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk,
                                 int dv, const void* q, const void* k, const void* v,
                                 const void* dout, const void* bias, void* out, void* dq,
                                 void* dk_out, void* dv_out, void* dbias);
/* asynchronous twin: returns once the step is enqueued (uploads, kernels and
 * downloads on separate streams); consecutive steps overlap one step's
 * downloads with the next one's uploads. Host buffers must stay untouched
 * until gte_ctx_sync(), which waits for every enqueued step. */
int gte_sparse_attn_fwd_bwd_host_async(gte_ctx* ctx, const gte_plan* plan, int dtype, int H, int dk,
                                 int dv, const void* q, const void* k, const void* v,
                                 const void* dout, const void* bias, void* out, void* dq,
                                 void* dk_out, void* dv_out, void* dbias);

/* ---- graph builders (device int32 CSR, bit-exact with the reference) ----
 * graph_from_edges   proj/src/graph.cpp:49-66  (range check -> DataError, sort, unique)
 * add_self_loops     proj/src/graph.cpp:127-149
 * permute_graph      proj/src/partition.cpp:435-456 (forward: host int64 old->new)
 * Output buffers: d_cols capacity m (graph_from_edges), nnz + n (add_self_loops),
 * nnz (permute_graph); row pointers n + 1. */
int gte_graph_from_edges(gte_ctx* ctx, int64_t n, int64_t m, const int32_t* d_src, const int32_t* d_dst,
                         int32_t* d_row_ptr, int32_t* d_cols, int64_t* nnz_out);
int gte_add_self_loops(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                       int32_t* d_out_row_ptr, int32_t* d_out_cols, int64_t* nnz_out);
int gte_permute_graph(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                      const int64_t* forward, int32_t* d_out_row_ptr, int32_t* d_out_cols);

/* ---- cluster-aware order (reference proj/src/partition.cpp) ----
 * gte_reorder: host CSR (int64, the reference Graph layout) -> Permutation;
 * bit-identical to gte::reorder(g, k, seed) (partition.cpp:413-433). Host-side
 * greedy (matching/FM/growth are sequential); see csrc/reorder.cpp. */
int gte_reorder(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t k, uint64_t seed,
                int64_t* forward, int64_t* inverse);
int gte_cluster_boundaries(int64_t n, int64_t k, int64_t* boundaries);
/* k x k cell histogram on the GPU; forward NULL = graph already in cluster
 * order. Outputs host arrays bnd[k+1], cell_nnz[k*k], cell_density[k*k]
 * (fp64, bit-exact: partition.cpp:514-539). */
int gte_build_cluster_grid(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                           const int64_t* forward, int64_t k, int64_t* bnd, int64_t* cell_nnz,
                           double* cell_density);
int gte_diagonal_edge_fraction(int64_t k, const int64_t* cell_nnz, double* out);

/* ---- Elastic Computation Reformation (reference proj/src/reformation.cpp) ----
 * gte_pack_subblocks: reformation.cpp:56-109, same tile sequence; tiles_rc
 * capacity 2*ceil(m/d_b^2).
 * gte_build_layout: reformation.cpp:111-195. g_perm (device CSR) must be in the
 * grid's cluster order. strategy 0 = Indolent (threshold beta_g), 1 = Elastic
 * (threshold beta_thre); Transferred iff cell_density < threshold (fp64). */
typedef struct gte_layout gte_layout;
int gte_pack_subblocks(int64_t m, const int64_t* er, const int64_t* ec, int64_t n_rows, int64_t n_cols,
                       int64_t d_b, int64_t* tiles_rc, int64_t* ntiles);
int gte_build_layout(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                     int64_t k, const int64_t* bnd, const int64_t* cell_nnz, const double* cell_density,
                     int strategy, double beta_thre, double beta_g, int64_t d_b, gte_layout** out);
int gte_layout_info(const gte_layout* L, int64_t* transferred_cells, int64_t* n_blocks, int64_t* dropped_edges,
                    int64_t* pattern_nnz);
int gte_layout_cells(const gte_layout* L, int32_t* cell_state, int64_t* block_off, int64_t* blocks);
int gte_layout_pattern_device(const gte_layout* L, const int32_t** d_row_ptr, const int32_t** d_cols);
int gte_layout_pattern_host(const gte_layout* L, int64_t* row_off, int64_t* cols);
int gte_layout_destroy(gte_layout* L);

/* Host-pointer twins of the builders (int64 reference CSR in host memory;
 * H2D, GPU build, D2H; synchronous). Capacities as for the device versions. */
int gte_graph_from_edges_host(gte_ctx* ctx, int64_t n, int64_t m, const int64_t* src, const int64_t* dst,
                              int64_t* row_off, int64_t* cols, int64_t* nnz_out);
int gte_add_self_loops_host(gte_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                            int64_t* out_row_off, int64_t* out_cols, int64_t* nnz_out);
int gte_permute_graph_host(gte_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                           const int64_t* forward, int64_t* out_row_off, int64_t* out_cols);
int gte_build_cluster_grid_host(gte_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                                const int64_t* forward, int64_t k, int64_t* bnd, int64_t* cell_nnz,
                                double* cell_density);
int gte_build_layout_host(gte_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                          int64_t k, const int64_t* bnd, const int64_t* cell_nnz, const double* cell_density,
                          int strategy, double beta_thre, double beta_g, int64_t d_b, gte_layout** out);

/* ---- host control logic (reference reformation.cpp:224-296,
 * interleave.cpp:68-106, parallel.cpp:96-113) ---- */
typedef struct gte_tuner gte_tuner;
int gte_tuner_create(double beta_g, int64_t delta, gte_tuner** out);
int gte_tuner_update(gte_tuner* st, double loss, double epoch_time_s, int64_t epoch);
int gte_tuner_state(const gte_tuner* st, double* avg_loss, int64_t* idx, double* thresholds, int64_t* n_thresholds,
                    int32_t* has_loss);
int gte_tuner_history(const gte_tuner* st, int64_t* epochs, double* ldr, int64_t* n);
int gte_tuner_set(gte_tuner* st, double avg_loss, int64_t idx, int32_t has_loss, int64_t n_hist,
                  const int64_t* epochs, const double* ldr);
int gte_tuner_load(gte_tuner* st, int64_t n_thresholds, const double* thresholds, int64_t delta);
int gte_tuner_destroy(gte_tuner* st);
int gte_select_k(int64_t l2_bytes, int64_t hidden_dim, int64_t i, int64_t* out);
int gte_select_db(int64_t n, const int64_t* db, const double* thr, int64_t* out);
/* flags[3] = {c1_self_attend, c2_pass, c3_reachable_within_l};
 * ints[4] = {layers, sweep_from, sweep_to, diameter_lower_bound} */
int gte_check_conditions(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t layers,
                         int32_t* flags, int64_t* ints);
int gte_select_mode(const int32_t* flags, int64_t epoch, int64_t dense_period, int32_t* mode, int32_t* reason);
int gte_partition_sequence(int64_t seq_len, int64_t num_workers, uint64_t seed, int64_t* ids, int64_t* padded);

/* ---- the transformer layer around the attention (reference
 * Trainer forward/backward, model.cpp:533-595, 669-744; LayerNorm
 * matrix.cpp:91-139, eps 1e-6; tanh GELU model.cpp:20-32) ----
 * One pre-LN GPH block on the device over a plan (pattern in h's row order):
 *   a = LN1(h); q,k,v = a W + b; attn = sparse attention (bias_vals [E]);
 *   h += attn W_o + b_o; u = LN2(h) W_ff1 + b_ff1; h += gelu(u) W_ff2 + b_ff2
 * Weights row-major [in x out] of dtype (X W); biases and LayerNorm scale /
 * shift in the accumulate type. The forward keeps its activations for the
 * backward, which ACCUMULATES parameter gradients (all in the accumulate
 * type) into `grads`, adds into dh in place, and writes the attention's
 * dbias_vals [E] (summed over heads). Projections are cuBLAS GEMMs; dropout
 * off. */
typedef struct gte_gph_params {
  void *ln1_scale, *ln1_shift, *w_q, *b_q, *w_k, *b_k, *w_v, *b_v, *w_o, *b_o;
  void *ln2_scale, *ln2_shift, *w_ff1, *b_ff1, *w_ff2, *b_ff2;
} gte_gph_params;
typedef struct gte_gph_layer gte_gph_layer;
int gte_gph_layer_create(gte_ctx* ctx, const gte_plan* plan, int dtype, int heads, int hidden, int ffn,
                         gte_gph_layer** out);
int gte_gph_layer_set_params(gte_gph_layer* layer, const gte_gph_params* params);
int gte_gph_layer_fwd(gte_gph_layer* layer, void* h, const void* bias_vals);
int gte_gph_layer_bwd(gte_gph_layer* layer, void* dh, const void* bias_vals, const gte_gph_params* grads,
                      void* dbias_vals);
int gte_gph_layer_destroy(gte_gph_layer* layer);

/* ---- ingestion formats (reference graph.cpp:68-109,
 * 302-336, partition.cpp:458-493), parsed from memory (the drop-in hands over
 * a std::istream's bytes); DataError with the reference's wording ----
 * gte_parse_edge_list: "src dst" per line, '#' comments; num_nodes_hint < 0
 *   = none (n = max id + 1, "empty graph" when no edge). Multi-threaded.
 *   The CSR comes from gte_graph_from_edges_host (GPU sort + unique).
 * gte_gtf1_decode: "GTF1", u64 N, u64 f, N*f float32; out = NULL reads the
 *   shape only. gte_gtf1_encode: out = NULL returns the byte length.
 * gte_parse_permutation: "old pos" per line; forward/inverse = NULL returns
 *   the size only. */
typedef struct gte_edges gte_edges;
int gte_parse_edge_list(const char* text, int64_t len, int64_t num_nodes_hint, gte_edges** out);
int gte_edges_info(const gte_edges* e, int64_t* num_nodes, int64_t* num_edges);
int gte_edges_copy(const gte_edges* e, int64_t* src, int64_t* dst);
int gte_edges_destroy(gte_edges* e);
int gte_gtf1_decode(const void* bytes, int64_t len, int64_t* n, int64_t* f, float* out);
int gte_gtf1_encode(int64_t n, int64_t f, const float* data, void* out, int64_t* len);
int gte_parse_permutation(const char* text, int64_t len, int64_t* n, int64_t* forward, int64_t* inverse);

/* ---- dense (all-pairs) attention, flash-style (reference attention.cpp:46-94,
 * 174-239; Trainer dense epochs model.cpp:395-405) ----
 * Rows r < s_real attend exactly the columns [0, s_real); pad rows r >= s_real
 * attend only themselves (out = m * v_r, no score gradient). s_real = S is the
 * reference's dense_attention. bias: [S x S] accumulate-type, shared by heads,
 * or null; wmult: head-major [H x S x S] or null; lse [S x H] (log2 units for
 * f32/bf16, natural log for f64); dbias [S x S] summed over heads, or null. */
int gte_dense_attn_fwd(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                       const void* k, int64_t ldq, const void* v, int64_t ldv, const void* bias, const void* wmult,
                       void* out, void* lse);
int gte_dense_attn_bwd(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                       const void* k, int64_t ldq, const void* v, int64_t ldv, const void* out, const void* lse,
                       const void* dout, const void* bias, const void* wmult, void* dq, void* dk_out, void* dv_out,
                       void* dbias);
/* Bucket-bias form of the Trainer's dense epoch (model.cpp:395-423, 520-523):
 * bias[r][c] = table[buckets[r][c]] with uint8 buckets [S x S] (execution
 * coordinates, gte_dense_buckets) and a table of n_buckets (<= 12) values of
 * the accumulate type; the backward returns the table's gradient dtable
 * [n_buckets] (dbias summed per bucket and over heads, fixed order) instead of
 * an S x S dbias. */
int gte_dense_attn_fwd_buckets(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv,
                               const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                               const uint8_t* buckets, const void* table, int64_t n_buckets, const void* wmult,
                               void* out, void* lse);
int gte_dense_attn_bwd_buckets(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv,
                               const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv, const void* out,
                               const void* lse, const void* dout, const uint8_t* buckets, const void* table,
                               int64_t n_buckets, const void* wmult, void* dq, void* dk_out, void* dv_out,
                               void* dtable);
/* gte_dense_buckets: the bucket matrix of a dense epoch (model.cpp:407-423):
 * rows r < s_real (execution coordinates) of d_out [S x S]: 0 self, 1 to/from
 * the global token (global_index, or -1), else the capped SPD of the original
 * nodes over the graph (max_dist + 1 beyond the cap), one BFS per row on the
 * device. perm forward [s_real], inverse [S] (int64, device). */
int gte_dense_buckets(gte_ctx* ctx, int64_t S, int64_t s_real, const int64_t* d_perm_forward,
                      const int64_t* d_perm_inverse, int64_t global_index, int64_t graph_n, int64_t graph_nnz,
                      const int32_t* d_graph_row_ptr, const int32_t* d_graph_cols, int64_t max_dist, uint8_t* d_out);
int gte_dense_attn_fwd_host(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                            const void* k, const void* v, const void* bias, const void* wmult, void* out, void* lse);
int gte_dense_attn_bwd_host(gte_ctx* ctx, int dtype, int64_t S, int64_t s_real, int H, int dk, int dv, const void* q,
                            const void* k, const void* v, const void* bias, const void* wmult, const void* dout,
                            void* dq, void* dk_out, void* dv_out, void* dbias);

/* ---- Trainer glue (reference model.cpp:76-83, 407-423, 447-463, 520-523) ----
 * extend_with_pad_loops: rows [rows, s_pad) get one self-loop each (host;
 * out_row_off [max(rows, s_pad) + 1], out_cols [nnz + max(0, s_pad - rows)]).
 * pattern_buckets: SPD bias bucket per attended pair, the Trainer's rule: 0
 * for the same token, 1 if either is the global token, max_dist + 1 if either
 * lies past the SPD table (pads) or the pair is absent from it, else its
 * distance (SpdTable::lookup, graph.cpp:208-214). The SPD table is the
 * reference's sparse CSR (row_off int64 [spd_n + 1], cols int64, dist uint16).
 * bias_from_table: bias[e] = table[bucket[e]]; dbias_to_table: the table's
 * gradient, summed in a fixed order (workspace: 296 * n_buckets floats). */
int gte_extend_with_pad_loops_host(int64_t rows, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                                   int64_t s_pad, int64_t* out_row_off, int64_t* out_cols);
int gte_pattern_buckets(gte_ctx* ctx, int64_t rows, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                        const int64_t* d_perm_inverse, int64_t global_index, int64_t spd_n,
                        const int64_t* d_spd_row_off, const int64_t* d_spd_cols, const uint16_t* d_spd_dist,
                        int64_t max_dist, int32_t* d_buckets);
int gte_bias_from_table(gte_ctx* ctx, int64_t nnz, const int32_t* d_buckets, const float* d_table, int64_t n_buckets,
                        float* d_bias);

/* ---- SPD buckets on the GPU (reference spd_table,
 * graph.cpp:208-261, without its N <= 20000 guard) ----
 * Graph: device int32 CSR of the reference Graph (arcs traversed both ways,
 * self loops ignored). Distances beyond max_dist (or unreachable) are
 * max_dist + 1 (SpdTable::unreachable_bucket).
 * gte_spd_table: the reference's table (rows = sources, columns ascending,
 *   uint16 distances <= max_dist), one capped BFS per source on the device;
 *   gte_spd_info / gte_spd_copy_host read it back (int64 row_off [n + 1],
 *   int64 cols, uint16 dist [total]).
 * gte_spd_pairs: distances of n_pairs (src, dst) pairs without the table
 *   (radius-2 balls + min-plus meet in the middle, early-exit BFS for the
 *   pairs beyond 4 hops); d_dist int32.
 * gte_pattern_buckets_graph: the Trainer's bucket per attended pair
 *   (model.cpp:447-463) with SPD from the graph itself: same rules as
 *   gte_pattern_buckets, lookup replaced by gte_spd_pairs. */
typedef struct gte_spd gte_spd;
int gte_spd_table(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                  int64_t max_dist, gte_spd** out);
int gte_spd_info(const gte_spd* t, int64_t* n, int64_t* max_dist, int64_t* total);
int gte_spd_copy_host(const gte_spd* t, int64_t* row_off, int64_t* cols, uint16_t* dist);
int gte_spd_destroy(gte_spd* t);
int gte_spd_pairs(gte_ctx* ctx, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                  int64_t max_dist, int64_t n_pairs, const int32_t* d_src, const int32_t* d_dst, int32_t* d_dist);
int gte_pattern_buckets_graph(gte_ctx* ctx, int64_t rows, int64_t nnz, const int32_t* d_row_ptr,
                              const int32_t* d_cols, const int64_t* d_perm_inverse, int64_t global_index,
                              int64_t graph_n, int64_t graph_nnz, const int32_t* d_graph_row_ptr,
                              const int32_t* d_graph_cols, int64_t max_dist, int32_t* d_buckets);
int gte_dbias_to_table(gte_ctx* ctx, int64_t nnz, const int32_t* d_buckets, const float* d_dbias, int64_t n_buckets,
                       float* d_table_grad, float* d_workspace);

/* ---- sequence parallelism (reference parallel.cpp:115-332, Ulysses
 * head-split all-to-all) ----
 * gte_sp: the exchange plan of P workers — token ids per worker (worker-major,
 * P x rows, the partition_sequence order; a permutation of [0, P*rows)) and the
 * cluster permutation's forward map (old -> execution position; null =
 * identity). The four halves of the two exchanges (d = hidden width, H =
 * heads for the divisibility checks of parallel.cpp:39-46, chunk = rows x d/P):
 *   pack_seq    worker shard [rows x d]   -> send [P][rows][d/P] (chunk p = columns p*d/P..)
 *   unpack_head recv [P][rows][d/P]       -> slice [S_pad x d/P], row of token t at perm.forward[t]
 *   pack_head   slice [S_pad x d/P]       -> send [P][rows][d/P] (chunk p = worker p's tokens)
 *   unpack_seq  recv [P][rows][d/P]       -> worker shard [rows x d] (chunk p -> columns p*d/P..)
 * The exchange between them is an equal-split all-to-all: gte_comm_all_to_all
 * (NCCL, one rank per GPU) or gte_sp_loopback (P logical workers in one
 * process, send_all [src][dst] -> recv_all [dst][src]). */
typedef struct gte_sp gte_sp;
typedef struct gte_comm gte_comm;
#define GTE_NCCL_ID_BYTES 128
int gte_sp_create(gte_ctx* ctx, int64_t P, int64_t rows_per_worker, const int64_t* token_ids,
                  const int64_t* perm_forward, gte_sp** out);
int gte_sp_destroy(gte_sp* sp);
int gte_sp_shape(const gte_sp* sp, int64_t* P, int64_t* rows_per_worker, int64_t* total);
int gte_sp_pack_seq(gte_ctx* ctx, const gte_sp* sp, int dtype, int64_t d, int64_t H, const void* shard, void* send);
int gte_sp_unpack_head(gte_ctx* ctx, const gte_sp* sp, int dtype, int64_t d, int64_t H, const void* recv,
                       void* slice_exec);
int gte_sp_pack_head(gte_ctx* ctx, const gte_sp* sp, int dtype, int64_t d, int64_t H, const void* slice_exec,
                     void* send);
int gte_sp_unpack_seq(gte_ctx* ctx, const gte_sp* sp, int dtype, int64_t d, int64_t H, const void* recv,
                      void* shard);
int gte_sp_loopback(gte_ctx* ctx, const gte_sp* sp, int dtype, int64_t d, const void* send_all, void* recv_all);
/* dbias of the distributed backward: sum of P per-worker partials [P][n] in
 * worker order (parallel.cpp:319); dtype selects f64 or f32 accumulators */
int gte_sp_ordered_sum(gte_ctx* ctx, int dtype, int64_t P, int64_t n, const void* parts, void* out);
/* NCCL communicator (one rank per GPU; the id comes from rank 0's
 * gte_nccl_unique_id, shared out of band, e.g. torch.distributed) */
int gte_nccl_unique_id(void* id_out);
int gte_comm_create(gte_ctx* ctx, int nranks, int rank, const void* id, gte_comm** out);
int gte_comm_destroy(gte_comm* comm);
int gte_comm_all_to_all(gte_comm* comm, gte_ctx* ctx, const void* send, void* recv, int64_t bytes_per_peer);
int gte_comm_all_gather(gte_comm* comm, gte_ctx* ctx, const void* send, void* recv, int64_t bytes);
/* variable all-to-all: per-peer byte offsets and counts (0 = no message) */
int gte_comm_all_to_allv(gte_comm* comm, gte_ctx* ctx, const void* send, const int64_t* send_off,
                         const int64_t* send_bytes, void* recv, const int64_t* recv_off, const int64_t* recv_bytes);
/* ---- the distributed layer as one object (SURVEY §8(b6) gte_sp_layer_fwd/bwd;
 * reference run_distributed_layer / run_distributed_layer_backward,
 * parallel.cpp:190-252, 271-332) ----
 * Built on a gte_sp (token ids + cluster permutation) and a plan (pattern in
 * execution coordinates, S_pad rows). comm == NULL: all P workers in this
 * process (the reference's in-process exchange); otherwise this process is
 * worker `rank` of a P-rank NCCL communicator. Shard arrays hold one device
 * pointer per local worker ([rows x d] each; P of them, or 1 with comm).
 * bias [E] and wmult [H x E] are in the accumulate type and replicated.
 * The backward reuses the forward's head slices and returns dbias summed
 * over workers in worker order (parallel.cpp:319). The ledger stays with the
 * caller (pure arithmetic: 4Sd/P per worker, parallel.cpp:83-94). */
typedef struct gte_sp_layer gte_sp_layer;
int gte_sp_layer_create(gte_ctx* ctx, const gte_sp* sp, const gte_plan* plan, gte_comm* comm, int rank, int dtype,
                        int64_t H, int64_t d, gte_sp_layer** out);
int gte_sp_layer_fwd(gte_sp_layer* layer, const void* const* q, const void* const* k, const void* const* v,
                     const void* bias, const void* wmult, void* const* out, int flags);
int gte_sp_layer_bwd(gte_sp_layer* layer, const void* const* dout, const void* bias, const void* wmult,
                     void* const* dq, void* const* dk, void* const* dv, void* dbias);
int gte_sp_layer_destroy(gte_sp_layer* layer);

/* ---- cluster-halo sequence parallelism ("Mode H") ----
 * Each GPU owns a contiguous range of rows (all heads) and runs the attention
 * kernels on a local plan over [own rows | halo rows]; the halo exchange moves
 * K/V rows of remote neighbours in (gather -> all_to_allv straight into the
 * halo tail) and the dK/dV partials of halo rows back to their owners
 * (all_to_allv -> scatter-add, peers in rank order). */
int gte_rows_gather(gte_ctx* ctx, int dtype, int64_t n, const int32_t* idx, const void* src, int64_t ld, int64_t w,
                    void* dst);
int gte_rows_scatter_add(gte_ctx* ctx, int dtype, int64_t n, const int32_t* idx, const void* src, int64_t w,
                         void* dst, int64_t ld);
/* All peers' partials in one launch: for u < n_rows, row rows[u] of dst gets
 * src rows pos[ptr[u]], pos[ptr[u] + 1], ... added one after the other, in
 * that order (the order of the per-peer gte_rows_scatter_add calls it
 * replaces, with the same per-add rounding: bit-identical). src rows are
 * ld_src apart, dst rows ld apart, w elements each. */
int gte_rows_scatter_add_seq(gte_ctx* ctx, int dtype, int64_t n_rows, const int32_t* rows, const int32_t* ptr,
                             const int32_t* pos, const void* src, int64_t ld_src, int64_t w, void* dst, int64_t ld);

#ifdef __cplusplus
}
#endif
#endif

/* gte_b200 — C ABI of the B200-native TorchGT graph-attention hot path.
 *
 * Plain pointers and sizes, no C++ or torch types. Every entry returns a
 * gte_status; on failure gte_last_error() holds a message whose wording
 * follows the reference exception it replaces, so the C++ drop-in layer
 * (include/gte/, csrc/gte_shim.cpp) can rethrow ConfigError/DataError with the
 * same substrings (reference error taxonomy: proj/include/gte/types.hpp:13-24).
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

enum { GTE_FORBID_EMPTY_ROWS = 1 };

typedef struct gte_ctx gte_ctx;
typedef struct gte_plan gte_plan;

const char* gte_last_error(void);
const char* gte_version(void);

/* ---- context: device, stream, workspaces, latched device errors ---- */
int gte_ctx_create(int device, gte_ctx** out);
int gte_ctx_destroy(gte_ctx* ctx);
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

#ifdef __cplusplus
}
#endif
#endif

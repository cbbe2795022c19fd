// Ulysses sequence-parallel attention layer behind one C-ABI object: the
// reference's run_distributed_layer / run_distributed_layer_backward
// (proj/src/parallel.cpp:190-252, 271-332) on device buffers, composed from
// the exchange halves of sp.cu and the sparse kernels (capi.cu):
//
//   fwd  Q, K, V shards --pack_seq--> a2a --unpack_head--> head slices
//        [S_pad x d/P] in execution coordinates (cluster permutation folded
//        into the unpack) -> sparse attention over the plan for the worker's
//        H/P heads -> pack_head --> a2a --> unpack_seq -> out shards.
//   bwd  dO shards -> head slices; the forward's cached Q/K/V/O/LSE slices
//        (the reference re-gathers them, :291-293 — same values) -> sparse
//        backward -> dQ/dK/dV back to shards; dbias = per-worker partials
//        summed in worker order (:319).
//
// Workers: with comm == NULL all P workers live in this process (the
// reference's in-process collective; exchange = gte_sp_loopback); with a
// gte_comm this process is worker `rank` of P (one per GPU; exchange = NCCL
// all-to-all, the dbias partials all-gathered before the ordered sum).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

namespace {

struct Buf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  ~Buf() { cudaFree(p); }
};

size_t esize(int dt) { return dt == GTE_F64 ? 8 : dt == GTE_F32 ? 4 : 2; }
size_t asize(int dt) { return dt == GTE_F64 ? 8 : 4; }
char* at(void* p, size_t off) { return static_cast<char*>(p) + off; }
const char* at(const void* p, size_t off) { return static_cast<const char*>(p) + off; }

#define LTRY(x)                \
  do {                         \
    int rc_ = (x);             \
    if (rc_) return rc_;       \
  } while (0)
#define LCUDA(x)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

struct gte_sp_layer {
  gte_ctx* ctx = nullptr;
  const gte_sp* sp = nullptr;
  const gte_plan* plan = nullptr;
  gte_comm* comm = nullptr;
  int dtype = GTE_F32;
  int64_t P = 0, rows = 0, H = 0, d = 0, hpw = 0, dh = 0, slice = 0, S = 0, E = 0, rank = 0, nlocal = 0;
  Buf send, recv;                             // exchange blocks
  std::vector<Buf> q, k, v, o, lse, up, dq, dk, dv;  // per local worker: head slices [S x slice], lse [S x hpw]
  Buf parts, gathered;                        // dbias partials [P][E]
  bool have_fwd = false;

  int64_t worker(int64_t w) const { return comm ? rank : w; }
  size_t chunk() const { return (size_t)rows * slice * esize(dtype); }  // one (src, dst) block

  // shards (one per local worker, [rows x d]) -> head slices `dst`
  int seq_to_head(const void* const* shards, std::vector<Buf>& dst) {
    const size_t block = chunk() * P;
    if (comm) {
      LCUDA(send.ensure(block));
      LCUDA(recv.ensure(block));
      LTRY(gte_sp_pack_seq(ctx, sp, dtype, d, H, shards[0], send.p));
      LTRY(gte_comm_all_to_all(comm, ctx, send.p, recv.p, (int64_t)chunk()));
      LCUDA(dst[0].ensure((size_t)S * slice * esize(dtype)));
      return gte_sp_unpack_head(ctx, sp, dtype, d, H, recv.p, dst[0].p);
    }
    LCUDA(send.ensure(block * P));
    LCUDA(recv.ensure(block * P));
    for (int64_t w = 0; w < P; ++w) LTRY(gte_sp_pack_seq(ctx, sp, dtype, d, H, shards[w], at(send.p, block * w)));
    LTRY(gte_sp_loopback(ctx, sp, dtype, d, send.p, recv.p));
    for (int64_t w = 0; w < P; ++w) {
      LCUDA(dst[w].ensure((size_t)S * slice * esize(dtype)));
      LTRY(gte_sp_unpack_head(ctx, sp, dtype, d, H, at(recv.p, block * w), dst[w].p));
    }
    return GTE_OK;
  }

  // head slices -> shards
  int head_to_seq(std::vector<Buf>& src, void* const* shards) {
    const size_t block = chunk() * P;
    if (comm) {
      LTRY(gte_sp_pack_head(ctx, sp, dtype, d, H, src[0].p, send.p));
      LTRY(gte_comm_all_to_all(comm, ctx, send.p, recv.p, (int64_t)chunk()));
      return gte_sp_unpack_seq(ctx, sp, dtype, d, H, recv.p, shards[0]);
    }
    for (int64_t w = 0; w < P; ++w) LTRY(gte_sp_pack_head(ctx, sp, dtype, d, H, src[w].p, at(send.p, block * w)));
    LTRY(gte_sp_loopback(ctx, sp, dtype, d, send.p, recv.p));
    for (int64_t w = 0; w < P; ++w) LTRY(gte_sp_unpack_seq(ctx, sp, dtype, d, H, at(recv.p, block * w), shards[w]));
    return GTE_OK;
  }

  const void* wm_of(const void* wmult, int64_t w) const {  // worker w's heads of [H][E] (parallel.cpp:239-243)
    return wmult ? at(wmult, (size_t)worker(w) * hpw * E * asize(dtype)) : nullptr;
  }
};

extern "C" {

int gte_sp_layer_create(gte_ctx* ctx, const gte_sp* sp, const gte_plan* plan, gte_comm* comm, int rank, int dtype,
                        int64_t H, int64_t d, gte_sp_layer** out) {
  int64_t P = 0, rows = 0, total = 0;
  LTRY(gte_sp_shape(sp, &P, &rows, &total));
  int64_t prow = 0, pnnz = 0;
  LTRY(gte_plan_shape(plan, &prow, &pnnz, nullptr, nullptr));
  if (prow != total) return set_error(GTE_CONFIG, "run_distributed_layer: pattern/sequence mismatch");
  if (H < 1 || H % P != 0) return set_error(GTE_CONFIG, "all_to_all: head count not divisible by worker count");
  if (d % H != 0) return set_error(GTE_CONFIG, "all_to_all: hidden dim not divisible by head count");
  if (comm && (rank < 0 || rank >= P)) return set_error(GTE_CONFIG, "run_distributed_layer: rank outside the workers");
  auto* L = new gte_sp_layer();
  L->ctx = ctx;
  L->sp = sp;
  L->plan = plan;
  L->comm = comm;
  L->dtype = dtype;
  L->P = P;
  L->rows = rows;
  L->S = total;
  L->H = H;
  L->d = d;
  L->hpw = H / P;
  L->dh = d / H;
  L->slice = d / P;
  L->E = pnnz;
  L->rank = rank;
  L->nlocal = comm ? 1 : P;
  for (auto* v : {&L->q, &L->k, &L->v, &L->o, &L->lse, &L->up, &L->dq, &L->dk, &L->dv}) v->resize(L->nlocal);
  *out = L;
  return GTE_OK;
}

int gte_sp_layer_destroy(gte_sp_layer* L) {
  delete L;
  return GTE_OK;
}

int gte_sp_layer_fwd(gte_sp_layer* L, const void* const* q, const void* const* k, const void* const* v,
                     const void* bias, const void* wmult, void* const* out, int flags) {
  LTRY(L->seq_to_head(q, L->q));
  LTRY(L->seq_to_head(k, L->k));
  LTRY(L->seq_to_head(v, L->v));
  for (int64_t w = 0; w < L->nlocal; ++w) {
    LCUDA(L->o[w].ensure((size_t)L->S * L->slice * esize(L->dtype)));
    LCUDA(L->lse[w].ensure((size_t)L->S * L->hpw * asize(L->dtype)));
    LTRY(gte_sparse_attn_fwd(L->ctx, L->plan, L->dtype, (int)L->hpw, (int)L->dh, (int)L->dh, L->q[w].p, L->k[w].p,
                             L->slice, L->v[w].p, L->slice, bias, L->wm_of(wmult, w), L->o[w].p, L->lse[w].p, flags));
  }
  LTRY(L->head_to_seq(L->o, out));
  L->have_fwd = true;
  return GTE_OK;
}

int gte_sp_layer_bwd(gte_sp_layer* L, const void* const* dout, const void* bias, const void* wmult, void* const* dq,
                     void* const* dk, void* const* dv, void* dbias) {
  if (!L->have_fwd) return set_error(GTE_CONFIG, "run_distributed_layer_backward: no forward on this layer");
  LTRY(L->seq_to_head(dout, L->up));
  const size_t part = (size_t)L->E * asize(L->dtype);
  LCUDA(L->parts.ensure(part * L->P));
  for (int64_t w = 0; w < L->nlocal; ++w) {
    for (auto* b : {&L->dq, &L->dk, &L->dv}) LCUDA((*b)[w].ensure((size_t)L->S * L->slice * esize(L->dtype)));
    LTRY(gte_sparse_attn_bwd(L->ctx, L->plan, L->dtype, (int)L->hpw, (int)L->dh, (int)L->dh, L->q[w].p, L->k[w].p,
                             L->slice, L->v[w].p, L->slice, L->o[w].p, L->lse[w].p, L->up[w].p, bias,
                             L->wm_of(wmult, w), L->dq[w].p, L->dk[w].p, L->dv[w].p,
                             at(L->parts.p, part * L->worker(w))));
  }
  LTRY(L->head_to_seq(L->dq, dq));
  LTRY(L->head_to_seq(L->dk, dk));
  LTRY(L->head_to_seq(L->dv, dv));
  if (dbias) {
    const void* all = L->parts.p;
    if (L->comm) {  // every rank's partial, in rank (= worker) order
      LCUDA(L->gathered.ensure(part * L->P));
      LTRY(gte_comm_all_gather(L->comm, L->ctx, at(L->parts.p, part * L->rank), L->gathered.p, (int64_t)part));
      all = L->gathered.p;
    }
    LTRY(gte_sp_ordered_sum(L->ctx, L->dtype, L->P, L->E, all, dbias));
  }
  return GTE_OK;
}

}  // extern "C"

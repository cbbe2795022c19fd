// Sequence parallelism on the device: the Ulysses (head-split) all-to-all of
// the reference's distributed attention layer (proj/src/parallel.cpp:115-332)
// and an NCCL communicator for one rank per GPU.
//
// The reference runs P logical workers in one process and moves rows with
// std::copy; here a worker is a GPU (or, for the single-process API mirror,
// a slot of a device buffer) and an exchange is
//
//   pack (one kernel)  ->  all-to-all of P equal chunks  ->  unpack (one kernel)
//
// with the cluster permutation folded into the unpack / pack of the head-
// sliced side: seq->head places token t's row directly at execution position
// perm.forward[t] (parallel.cpp:48-55 permute_rows after :137-139), head->seq
// reads it back from there (unpermute_rows, :57-64, then :174-176). A chunk
// (src -> dst) is rows_per_worker x d/P elements, so the exchange is a plain
// equal-split all-to-all: ncclSend/ncclRecv pairs in one group over NVLink.
//
// Ledger (CommLedger, parallel.hpp:23-44) is exact host arithmetic in the
// Python mirror (paper_2407_14106_b200/parallel.py).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
int ctx_device(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define SCUDA(expr)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                 \
  } while (0)

#define SNCCL(expr)                                                                                    \
  do {                                                                                                 \
    ncclResult_t r_ = (expr);                                                                          \
    if (r_ != ncclSuccess)                                                                             \
      return set_error(GTE_NCCL, std::string("NCCL error: ") + nccl().GetErrorString(r_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                  \
  } while (0)

struct gte_sp {
  int64_t P = 0, rows = 0, total = 0;  // rows per worker, S_pad = P * rows
  int32_t* d_tokens = nullptr;          // [P * rows] token ids, worker-major (partition_sequence order)
  int32_t* d_pos = nullptr;             // [P * rows] execution position perm.forward[token]
};

// NCCL is resolved at first use with dlopen("libnccl.so.2"): inside a torch
// process that returns the NCCL torch already loaded (one NCCL per process),
// elsewhere the system library. Linking it at build time would pin the
// system NCCL into every process that loads libgte_b200.so first.
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("NCCL not found: ") + dlerror();
      return a;
    }
#define GTE_SYM(F) a.F = reinterpret_cast<decltype(a.F)>(dlsym(h, "nccl" #F))
    GTE_SYM(GetUniqueId);
    GTE_SYM(CommInitRank);
    GTE_SYM(CommDestroy);
    GTE_SYM(GroupStart);
    GTE_SYM(GroupEnd);
    GTE_SYM(Send);
    GTE_SYM(Recv);
    GTE_SYM(AllGather);
    GTE_SYM(GetErrorString);
#undef GTE_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv &&
           a.AllGather && a.GetErrorString;
    if (!a.ok) a.why = "NCCL library lacks a required symbol";
    return a;
  }();
  return api;
}
}  // namespace

#define NCCL_API_OR_FAIL()                                       \
  do {                                                           \
    if (!nccl().ok) return set_error(GTE_NCCL, nccl().why);      \
  } while (0)

struct gte_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

namespace {

unsigned blocks_for(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)g;
}

// Element unit of a row copy: 16, 8, 4 or 2 bytes (the widest dividing the
// chunk row and every pointer alignment).
template <typename U>
__global__ void pack_seq_kernel(const U* __restrict__ shard, U* __restrict__ send, int64_t rows, int64_t P,
                                int64_t nu) {
  // send[dst][r][0..nu) = shard[r][dst*nu .. (dst+1)*nu)
  const int64_t n = P * rows * nu;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x % nu, r = (x / nu) % rows, dst = x / (nu * rows);
    send[x] = shard[r * (P * nu) + dst * nu + c];
  }
}

template <typename U>
__global__ void unpack_head_kernel(const U* __restrict__ recv, U* __restrict__ slice, const int32_t* __restrict__ pos,
                                   int64_t rows, int64_t P, int64_t nu) {
  // recv[src][r] holds token tokens[src][r]: slice[pos[src*rows + r]] = recv[src][r]
  const int64_t n = P * rows * nu;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x % nu, sr = x / nu;
    slice[(int64_t)__ldg(pos + sr) * nu + c] = recv[x];
  }
}

template <typename U>
__global__ void pack_head_kernel(const U* __restrict__ slice, U* __restrict__ send, const int32_t* __restrict__ pos,
                                 int64_t rows, int64_t P, int64_t nu) {
  // send[dst][r] = slice[pos[dst*rows + r]]  (dst's tokens, in dst's shard order)
  const int64_t n = P * rows * nu;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x % nu, dr = x / nu;
    send[x] = slice[(int64_t)__ldg(pos + dr) * nu + c];
  }
}

template <typename U>
__global__ void unpack_seq_kernel(const U* __restrict__ recv, U* __restrict__ shard, int64_t rows, int64_t P,
                                  int64_t nu) {
  // shard[r][src*nu .. ) = recv[src][r]
  const int64_t n = P * rows * nu;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x % nu, r = (x / nu) % rows, src = x / (nu * rows);
    shard[r * (P * nu) + src * nu + c] = recv[x];
  }
}

template <typename A>
__global__ void ordered_sum_kernel(const A* __restrict__ parts, A* __restrict__ out, int64_t P, int64_t n) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    A s = parts[x];
    for (int64_t w = 1; w < P; ++w) s += parts[w * n + x];  // worker order (parallel.cpp:319)
    out[x] = s;
  }
}

// Cluster-halo exchange (Mode H): rows picked by an index list into a
// contiguous send block, and received partial rows added into their owner
// rows (one source at a time, rows unique per source: no atomics).
template <typename U>
__global__ void gather_rows_kernel(const U* __restrict__ src, int64_t ld, const int32_t* __restrict__ idx, int64_t n,
                                   int64_t nu, U* __restrict__ dst) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n * nu; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = x / nu, c = x % nu;
    dst[x] = src[(int64_t)__ldg(idx + r) * ld + c];
  }
}

template <typename T, typename A>
__global__ void scatter_add_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                                        int64_t w, T* __restrict__ dst, int64_t ld) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n * w; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = x / w, c = x % w;
    T* d = dst + (int64_t)__ldg(idx + r) * ld + c;
    *d = T(A(*d) + A(src[x]));
  }
}

// dst[rows[u]][c] += src[pos[j]][c] for j in [ptr[u], ptr[u+1]), in j order,
// rounding to T after every add (as the per-source kernel above does)
template <typename T, typename A>
__global__ void scatter_add_seq_kernel(const T* __restrict__ src, int64_t lds, const int32_t* __restrict__ rows,
                                       const int32_t* __restrict__ ptr, const int32_t* __restrict__ pos, int64_t n,
                                       int64_t w, T* __restrict__ dst, int64_t ld) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n * w; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = x / w, c = x % w;
    T* d = dst + (int64_t)__ldg(rows + u) * ld + c;
    T acc = *d;
    for (int j = __ldg(ptr + u), j1 = __ldg(ptr + u + 1); j < j1; ++j)
      acc = T(A(acc) + A(src[(int64_t)__ldg(pos + j) * lds + c]));
    *d = acc;
  }
}

int unit_bytes(int64_t chunk_row_bytes, std::initializer_list<const void*> ptrs) {
  for (int u : {16, 8, 4, 2, 1}) {
    if (chunk_row_bytes % u) continue;
    bool ok = true;
    for (const void* p : ptrs) ok = ok && (reinterpret_cast<uintptr_t>(p) % u == 0);
    if (ok) return u;
  }
  return 1;
}

size_t esize(int dtype) { return dtype == GTE_F64 ? 8 : dtype == GTE_F32 ? 4 : 2; }

// op: 0 pack_seq, 1 unpack_head, 2 pack_head, 3 unpack_seq
template <typename U>
void launch_op(int op, const void* in, void* out, const int32_t* pos, int64_t rows, int64_t P, int64_t nu,
               cudaStream_t st) {
  const unsigned g = blocks_for(P * rows * nu);
  const U* a = static_cast<const U*>(in);
  U* b = static_cast<U*>(out);
  switch (op) {
    case 0: pack_seq_kernel<U><<<g, 256, 0, st>>>(a, b, rows, P, nu); break;
    case 1: unpack_head_kernel<U><<<g, 256, 0, st>>>(a, b, pos, rows, P, nu); break;
    case 2: pack_head_kernel<U><<<g, 256, 0, st>>>(a, b, pos, rows, P, nu); break;
    default: unpack_seq_kernel<U><<<g, 256, 0, st>>>(a, b, rows, P, nu); break;
  }
}

int run_op(gte_ctx* ctx, const gte_sp* s, int op, int dtype, int64_t d, const void* in, void* out) {
  const int64_t cb = d / s->P * (int64_t)esize(dtype);  // bytes of one chunk row
  const int ub = unit_bytes(cb, {in, out});
  const int64_t nu = cb / ub;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  switch (ub) {
    case 16: launch_op<uint4>(op, in, out, s->d_pos, s->rows, s->P, nu, st); break;
    case 8: launch_op<uint2>(op, in, out, s->d_pos, s->rows, s->P, nu, st); break;
    case 4: launch_op<uint32_t>(op, in, out, s->d_pos, s->rows, s->P, nu, st); break;
    case 2: launch_op<uint16_t>(op, in, out, s->d_pos, s->rows, s->P, nu, st); break;
    default: launch_op<uint8_t>(op, in, out, s->d_pos, s->rows, s->P, nu, st); break;
  }
  ctx_launch_counter(ctx) += 1;
  SCUDA(cudaGetLastError());
  return GTE_OK;
}

// checks shared by the four exchange halves (parallel.cpp:39-46)
int sp_check(const gte_sp* s, int dtype, int64_t d, int64_t H) {
  if (!s) return set_error(GTE_CONFIG, "all_to_all: null plan");
  if (dtype != GTE_F64 && dtype != GTE_F32 && dtype != GTE_BF16) return set_error(GTE_CONFIG, "all_to_all: bad dtype");
  if (H > 0 && H % s->P != 0) return set_error(GTE_CONFIG, "all_to_all: head count not divisible by worker count");
  if (H > 0 && d % H != 0) return set_error(GTE_CONFIG, "all_to_all: hidden dim not divisible by head count");
  if (d < 1 || d % s->P != 0) return set_error(GTE_CONFIG, "all_to_all: hidden dim not divisible by head count");
  return GTE_OK;
}

}  // namespace

extern "C" {

int gte_sp_create(gte_ctx* ctx, int64_t P, int64_t rows_per_worker, const int64_t* token_ids,
                  const int64_t* perm_forward, gte_sp** out) {
  if (P < 1) return set_error(GTE_CONFIG, "partition_sequence: worker count must be >= 1");
  if (rows_per_worker < 1) return set_error(GTE_CONFIG, "all_to_all: empty shards");
  const int64_t total = P * rows_per_worker;
  if (total >= (int64_t(1) << 31)) return set_error(GTE_CONFIG, "all_to_all: sequence exceeds int32 range");
  std::vector<int32_t> tok(total), pos(total);
  std::vector<char> seen(total, 0);
  for (int64_t x = 0; x < total; ++x) {
    const int64_t t = token_ids[x];
    if (t < 0 || t >= total || seen[t]) return set_error(GTE_CONFIG, "all_to_all: token ids are not a permutation of [0, S_pad)");
    seen[t] = 1;
    const int64_t f = perm_forward ? perm_forward[t] : t;
    if (f < 0 || f >= total) return set_error(GTE_CONFIG, "run_distributed_layer: permutation size mismatch");
    tok[x] = (int32_t)t;
    pos[x] = (int32_t)f;
  }
  auto* s = new gte_sp();
  s->P = P;
  s->rows = rows_per_worker;
  s->total = total;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  if (cudaMalloc(&s->d_tokens, sizeof(int32_t) * total) != cudaSuccess ||
      cudaMalloc(&s->d_pos, sizeof(int32_t) * total) != cudaSuccess) {
    cudaFree(s->d_tokens);
    delete s;
    return set_error(GTE_CUDA, "sp: device allocation failed");
  }
  cudaMemcpyAsync(s->d_tokens, tok.data(), sizeof(int32_t) * total, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(s->d_pos, pos.data(), sizeof(int32_t) * total, cudaMemcpyHostToDevice, st);
  SCUDA(cudaStreamSynchronize(st));
  *out = s;
  return GTE_OK;
}

int gte_sp_shape(const gte_sp* s, int64_t* P, int64_t* rows_per_worker, int64_t* total) {
  if (!s) return set_error(GTE_CONFIG, "all_to_all: null plan");
  if (P) *P = s->P;
  if (rows_per_worker) *rows_per_worker = s->rows;
  if (total) *total = s->total;
  return GTE_OK;
}

int gte_sp_destroy(gte_sp* s) {
  if (!s) return GTE_OK;
  cudaFree(s->d_tokens);
  cudaFree(s->d_pos);
  delete s;
  return GTE_OK;
}

int gte_sp_pack_seq(gte_ctx* ctx, const gte_sp* s, int dtype, int64_t d, int64_t H, const void* shard, void* send) {
  int rc = sp_check(s, dtype, d, H);
  return rc ? rc : run_op(ctx, s, 0, dtype, d, shard, send);
}

int gte_sp_unpack_head(gte_ctx* ctx, const gte_sp* s, int dtype, int64_t d, int64_t H, const void* recv,
                       void* slice_exec) {
  int rc = sp_check(s, dtype, d, H);
  return rc ? rc : run_op(ctx, s, 1, dtype, d, recv, slice_exec);
}

int gte_sp_pack_head(gte_ctx* ctx, const gte_sp* s, int dtype, int64_t d, int64_t H, const void* slice_exec,
                     void* send) {
  int rc = sp_check(s, dtype, d, H);
  return rc ? rc : run_op(ctx, s, 2, dtype, d, slice_exec, send);
}

int gte_sp_unpack_seq(gte_ctx* ctx, const gte_sp* s, int dtype, int64_t d, int64_t H, const void* recv, void* shard) {
  int rc = sp_check(s, dtype, d, H);
  return rc ? rc : run_op(ctx, s, 3, dtype, d, recv, shard);
}

int gte_sp_loopback(gte_ctx* ctx, const gte_sp* s, int dtype, int64_t d, const void* send_all, void* recv_all) {
  // single-process exchange of P logical workers: send_all[src][dst] (chunks of
  // rows x d/P) -> recv_all[dst][src]; one 2-D copy per source worker
  if (!s) return set_error(GTE_CONFIG, "all_to_all: null plan");
  const size_t chunk = (size_t)s->rows * (size_t)(d / s->P) * esize(dtype);
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  for (int64_t src = 0; src < s->P; ++src) {
    // rows: dst; source pitch = chunk (consecutive dst chunks of src), destination pitch = P * chunk
    SCUDA(cudaMemcpy2DAsync(static_cast<char*>(recv_all) + src * chunk, s->P * chunk,
                            static_cast<const char*>(send_all) + src * s->P * chunk, chunk, chunk, (size_t)s->P,
                            cudaMemcpyDeviceToDevice, st));
  }
  return GTE_OK;
}

int gte_sp_ordered_sum(gte_ctx* ctx, int dtype, int64_t P, int64_t n, const void* parts, void* out) {
  // dbias = sum over workers in worker order (parallel.cpp:319); parts [P][n]
  if (P < 1 || n < 0) return set_error(GTE_CONFIG, "ordered_sum: bad sizes");
  if (n == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  if (dtype == GTE_F64)
    ordered_sum_kernel<double><<<blocks_for(n), 256, 0, st>>>(static_cast<const double*>(parts), static_cast<double*>(out), P, n);
  else
    ordered_sum_kernel<float><<<blocks_for(n), 256, 0, st>>>(static_cast<const float*>(parts), static_cast<float*>(out), P, n);
  ctx_launch_counter(ctx) += 1;
  SCUDA(cudaGetLastError());
  return GTE_OK;
}

int gte_rows_gather(gte_ctx* ctx, int dtype, int64_t n, const int32_t* idx, const void* src, int64_t ld, int64_t w,
                    void* dst) {
  // dst[r][0..w) = src[idx[r]][0..w), elements of `dtype`; dst dense (ld = w)
  if (n < 0 || w < 0 || ld < w) return set_error(GTE_CONFIG, "rows_gather: bad sizes");
  if (n == 0 || w == 0) return GTE_OK;
  const int64_t es = (int64_t)esize(dtype), rb = w * es;
  int ub = 16;
  while (ub > 1 && (rb % ub || (ld * es) % ub || reinterpret_cast<uintptr_t>(src) % ub ||
                    reinterpret_cast<uintptr_t>(dst) % ub))
    ub >>= 1;
  const int64_t nu = rb / ub, ldu = ld * es / ub;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const unsigned g = blocks_for(n * nu);
  switch (ub) {
    case 16: gather_rows_kernel<uint4><<<g, 256, 0, st>>>((const uint4*)src, ldu, idx, n, nu, (uint4*)dst); break;
    case 8: gather_rows_kernel<uint2><<<g, 256, 0, st>>>((const uint2*)src, ldu, idx, n, nu, (uint2*)dst); break;
    case 4: gather_rows_kernel<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)src, ldu, idx, n, nu, (uint32_t*)dst); break;
    case 2: gather_rows_kernel<uint16_t><<<g, 256, 0, st>>>((const uint16_t*)src, ldu, idx, n, nu, (uint16_t*)dst); break;
    default: gather_rows_kernel<uint8_t><<<g, 256, 0, st>>>((const uint8_t*)src, ldu, idx, n, nu, (uint8_t*)dst); break;
  }
  ctx_launch_counter(ctx) += 1;
  SCUDA(cudaGetLastError());
  return GTE_OK;
}

int gte_rows_scatter_add(gte_ctx* ctx, int dtype, int64_t n, const int32_t* idx, const void* src, int64_t w,
                         void* dst, int64_t ld) {
  // dst[idx[r]][0..w) += src[r][0..w) (accumulated in f32 for bf16); idx unique
  if (n < 0 || w < 0 || ld < w) return set_error(GTE_CONFIG, "rows_scatter_add: bad sizes");
  if (n == 0 || w == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const unsigned g = blocks_for(n * w);
  switch (dtype) {
    case GTE_F64:
      scatter_add_rows_kernel<double, double><<<g, 256, 0, st>>>((const double*)src, idx, n, w, (double*)dst, ld);
      break;
    case GTE_F32:
      scatter_add_rows_kernel<float, float><<<g, 256, 0, st>>>((const float*)src, idx, n, w, (float*)dst, ld);
      break;
    default:
      scatter_add_rows_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>((const __nv_bfloat16*)src, idx, n, w,
                                                                        (__nv_bfloat16*)dst, ld);
      break;
  }
  ctx_launch_counter(ctx) += 1;
  SCUDA(cudaGetLastError());
  return GTE_OK;
}

int gte_rows_scatter_add_seq(gte_ctx* ctx, int dtype, int64_t n, const int32_t* rows, const int32_t* ptr,
                             const int32_t* pos, const void* src, int64_t lds, int64_t w, void* dst, int64_t ld) {
  if (n < 0 || w < 0 || ld < w || lds < w) return set_error(GTE_CONFIG, "rows_scatter_add_seq: bad sizes");
  if (n == 0 || w == 0) return GTE_OK;
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const unsigned g = blocks_for(n * w);
  switch (dtype) {
    case GTE_F64:
      scatter_add_seq_kernel<double, double><<<g, 256, 0, st>>>((const double*)src, lds, rows, ptr, pos, n, w,
                                                                 (double*)dst, ld);
      break;
    case GTE_F32:
      scatter_add_seq_kernel<float, float><<<g, 256, 0, st>>>((const float*)src, lds, rows, ptr, pos, n, w,
                                                               (float*)dst, ld);
      break;
    default:
      scatter_add_seq_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>((const __nv_bfloat16*)src, lds, rows, ptr, pos,
                                                                       n, w, (__nv_bfloat16*)dst, ld);
      break;
  }
  ctx_launch_counter(ctx) += 1;
  SCUDA(cudaGetLastError());
  return GTE_OK;
}

// ---- NCCL: one rank per GPU over NVLink / NVSwitch ----
int gte_nccl_unique_id(void* id_out) {
  NCCL_API_OR_FAIL();
  ncclUniqueId id;
  SNCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == GTE_NCCL_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof id);
  return GTE_OK;
}

int gte_comm_create(gte_ctx* ctx, int nranks, int rank, const void* id_in, gte_comm** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(GTE_CONFIG, "comm: bad rank / world size");
  NCCL_API_OR_FAIL();
  // ncclCommInitRank binds the communicator to the calling thread's device:
  // make that the context's GPU (one rank per GPU)
  if (ctx) {
    const cudaError_t e = cudaSetDevice(ctx_device(ctx));
    if (e != cudaSuccess) return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
  }
  ncclUniqueId id;
  memcpy(&id, id_in, sizeof id);
  auto* c = new gte_comm();
  ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_error(GTE_NCCL, std::string("NCCL error: ") + nccl().GetErrorString(r) + " (ncclCommInitRank)");
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return GTE_OK;
}

int gte_comm_destroy(gte_comm* c) {
  if (!c) return GTE_OK;
  if (nccl().ok) nccl().CommDestroy(c->comm);
  delete c;
  return GTE_OK;
}

int gte_comm_all_to_all(gte_comm* c, gte_ctx* ctx, const void* send, void* recv, int64_t bytes_per_peer) {
  // equal-split all-to-all: chunk p of `send` goes to rank p, chunk p of `recv` comes from rank p
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const NcclApi& N = nccl();
  SNCCL(N.GroupStart());
  for (int p = 0; p < c->nranks; ++p) {
    SNCCL(N.Send(static_cast<const char*>(send) + p * bytes_per_peer, (size_t)bytes_per_peer, ncclUint8, p, c->comm, st));
    SNCCL(N.Recv(static_cast<char*>(recv) + p * bytes_per_peer, (size_t)bytes_per_peer, ncclUint8, p, c->comm, st));
  }
  SNCCL(N.GroupEnd());
  return GTE_OK;
}

int gte_comm_all_to_allv(gte_comm* c, gte_ctx* ctx, const void* send, const int64_t* send_off,
                         const int64_t* send_bytes, void* recv, const int64_t* recv_off, const int64_t* recv_bytes) {
  // variable all-to-all (byte offsets / counts per peer); zero-byte pairs skipped
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  const NcclApi& N = nccl();
  SNCCL(N.GroupStart());
  for (int p = 0; p < c->nranks; ++p) {
    if (send_bytes[p] > 0)
      SNCCL(N.Send(static_cast<const char*>(send) + send_off[p], (size_t)send_bytes[p], ncclUint8, p, c->comm, st));
    if (recv_bytes[p] > 0)
      SNCCL(N.Recv(static_cast<char*>(recv) + recv_off[p], (size_t)recv_bytes[p], ncclUint8, p, c->comm, st));
  }
  SNCCL(N.GroupEnd());
  return GTE_OK;
}

int gte_comm_all_gather(gte_comm* c, gte_ctx* ctx, const void* send, void* recv, int64_t bytes) {
  cudaStream_t st = (cudaStream_t)ctx_stream(ctx);
  SNCCL(nccl().AllGather(send, recv, (size_t)bytes, ncclUint8, c->comm, st));
  return GTE_OK;
}

}  // extern "C"

// C ABI of the B200 graph-attention library (include/gte_b200.h): context,
// device pattern plans (CSR + CSC built on the GPU with radix sort/scan), and
// the sparse attention entries with their host-pointer twins.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <initializer_list>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/gte_b200.h"
#include "ecr_tile.cuh"
#include "tile_launch.cuh"

using namespace gte_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " \
                                + __FILE__ + ":" + std::to_string(__LINE__));            \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

size_t elem_size(int dtype) { return dtype == GTE_F64 ? 8 : dtype == GTE_F32 ? 4 : 2; }
size_t acc_size(int dtype) { return dtype == GTE_F64 ? 8 : 4; }

__global__ void expand_rows_kernel(const int32_t* __restrict__ row_ptr, int64_t rows,
                                   int32_t* __restrict__ row_of_edge) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int b = row_ptr[w], e = row_ptr[w + 1];
  for (int i = b + lane; i < e; i += 32) row_of_edge[i] = (int32_t)w;
}

__global__ void count_cols_kernel(const int32_t* __restrict__ cols, int64_t nnz, int32_t* counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + cols[i], 1);
}

__global__ void gather_rows_kernel(const int32_t* __restrict__ eid, const int32_t* __restrict__ row_of_edge,
                                   int64_t nnz, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = row_of_edge[eid[i]];
}

__global__ void iota_kernel(int32_t* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

__global__ void unref_kernel(const int32_t* __restrict__ counts, int64_t rows, int32_t* out, int32_t* n_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    if (counts[i] == 0) out[atomicAdd(n_out, 1)] = (int32_t)i;
}

__global__ void degree_kernel(const int32_t* __restrict__ ptr, int64_t rows, int32_t* deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = ptr[i + 1] - ptr[i];
}

__global__ void check_csr_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
                                 int64_t rows, int64_t nnz, int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    if (cols[i] < 0 || cols[i] >= rows) atomicOr(bad, 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    if (row_ptr[i + 1] < row_ptr[i]) atomicOr(bad, 2);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (row_ptr[0] != 0 || row_ptr[rows] != nnz)) atomicOr(bad, 2);
}

unsigned grid_for(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)g;
}

}  // namespace

struct gte_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;          // host->device copies of the *_host entries (lazy)
  cudaStream_t down = nullptr;          // device->host copies (lazy; its own copy engine direction)
  cudaEvent_t ev[8] = {};               // [0] inputs in, [1] dO in, [2] O ready, [3] grads ready,
                                        // [4] O read back, [5] grads read back, [6] scratch
  bool pending = false;                 // a previous fwd_bwd_host step is still in flight
  // double-buffered device sets of fwd_bwd_host (inputs + outputs), alternated
  // per step so one step's uploads and downloads overlap the other's kernels:
  // [0] q [1] k [2] v [3] out [4] lse [5] dbias [6] bias [7] dq [8] dk [9] dO [10] dv
  DevBuf hs[2][11];
  cudaEvent_t k_done[2] = {}, d2h_done[2] = {};
  bool hs_used[2] = {false, false};
  int parity = 0;
  int* d_err = nullptr;  // [0] non-finite bits, [1] first empty row
  int* h_err = nullptr;  // pinned mirror
  int64_t launches = 0;
  DevBuf io[13];  // [11] delta (generic), [12] packed (lse, delta) (tile)
  DevBuf scratch;  // workspace of other translation units (ctx_scratch)
};

namespace gte_b200 {
bool ecr_eligible(int H, int dk, int dv);
cudaError_t launch_ecr_bf16(bool bwd, const EcrArgs& a, cudaStream_t st);
}  // namespace gte_b200

// ECR split of a plan (gte_plan_set_blocks): dense 16 x 16 sub-blocks on the
// tensor pipe (ecr_tile.cuh) + the remainder pattern on the sparse kernels.
struct EcrSplit {
  int64_t n_blocks = 0, n_inc = 0, n_cinc = 0;
  int32_t* dev = nullptr;  // one allocation: blk, ebase, inc, cinc, inc_ptr, cinc_ptr, eid
  const int32_t *blk = nullptr, *ebase = nullptr, *inc = nullptr, *cinc = nullptr;
  const int32_t *inc_ptr = nullptr, *cinc_ptr = nullptr, *eid = nullptr;
  gte_plan* rem = nullptr;
  DevBuf part;  // tile partials (forward: (m, l) + acc; backward: dQ, dK, dV)
};

struct gte_plan {
  gte_ctx* ctx = nullptr;
  int64_t rows = 0, nnz = 0, max_row_deg = 0, max_col_deg = 0, n_unref = 0;
  int32_t* row_ptr = nullptr;
  int32_t* cols = nullptr;
  int32_t* col_ptr = nullptr;
  int32_t* csc_row = nullptr;
  int32_t* csc_eid = nullptr;
  int32_t* unref = nullptr;
  // execution plan of the tile kernels (build_exec): per pass the order of the
  // non-hub rows (columns), tile boundaries into it, and the hub list
  int32_t* exec = nullptr;  // one allocation holding the six arrays below
  const int32_t *order = nullptr, *tiles = nullptr, *hubs = nullptr;
  const int32_t *order_c = nullptr, *tiles_c = nullptr, *hubs_c = nullptr;
  int n_tiles = 0, n_hubs = 0, n_tiles_c = 0, n_hubs_c = 0;
  bool scheduled = false;
  int64_t communities = 0;
  std::vector<int64_t> host_order;  // execution order given to gte_plan_set_order (empty: natural)
  int64_t out_rows = -1;            // gte_plan_set_output_rows: the CSR pass skips rows >= out_rows
  EcrSplit* ecr = nullptr;
};

namespace {

int reset_err(gte_ctx* c) {
  const int init[2] = {0, INT_MAX};
  CUDA_TRY(cudaMemcpyAsync(c->d_err, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
  return GTE_OK;
}

// Reads the latched device errors (synchronising), maps them to the
// reference's DataError messages (proj/src/attention.cpp:20-22, 119-123).
int drain_errors(gte_ctx* c, bool ignore_nonfinite = false) {
  CUDA_TRY(cudaMemcpyAsync(c->h_err, c->d_err, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int bits = ignore_nonfinite ? 0 : c->h_err[0], row = c->h_err[1];
  if (c->h_err[0] == 0 && row == INT_MAX) return GTE_OK;
  int rc = reset_err(c);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (bits == 0 && row == INT_MAX) return GTE_OK;
  if (bits & 1) return fail(GTE_DATA, "attention: non-finite Q");
  if (bits & 2) return fail(GTE_DATA, "attention: non-finite K");
  if (bits & 4) return fail(GTE_DATA, "attention: non-finite V");
  return fail(GTE_DATA, "sparse_attention: row " + std::to_string(row) +
                            " attends to nothing; run add_self_loops");
}

int build_plan_device(gte_ctx* c, gte_plan* p) {
  const int64_t rows = p->rows, nnz = p->nnz;
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMallocAsync(&p->col_ptr, sizeof(int32_t) * (rows + 1), st));
  CUDA_TRY(cudaMallocAsync(&p->csc_row, sizeof(int32_t) * (nnz + 1), st));
  CUDA_TRY(cudaMallocAsync(&p->csc_eid, sizeof(int32_t) * (nnz + 1), st));
  CUDA_TRY(cudaMallocAsync(&p->unref, sizeof(int32_t) * (rows + 1), st));
  int32_t *row_of_edge = nullptr, *iota = nullptr, *sorted_cols = nullptr, *counts = nullptr, *scratch = nullptr;
  CUDA_TRY(cudaMallocAsync(&row_of_edge, sizeof(int32_t) * (nnz + 1), st));
  CUDA_TRY(cudaMallocAsync(&iota, sizeof(int32_t) * (nnz + 1), st));
  CUDA_TRY(cudaMallocAsync(&sorted_cols, sizeof(int32_t) * (nnz + 1), st));
  CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (rows + 2), st));
  CUDA_TRY(cudaMallocAsync(&scratch, sizeof(int32_t) * 4, st));
  CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (rows + 2), st));
  CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(int32_t) * 4, st));

  // validate before any kernel indexes with the pattern: an out-of-range
  // column or a non-monotone offset must come back as ConfigError, not as a
  // scatter out of bounds (sticky context error)
  check_csr_kernel<<<grid_for(nnz > rows ? nnz : rows), 256, 0, st>>>(p->row_ptr, p->cols, rows, nnz, scratch);
  {
    int32_t bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, scratch, sizeof bad, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (bad) {
      for (void* x : {(void*)row_of_edge, (void*)iota, (void*)sorted_cols, (void*)counts, (void*)scratch})
        cudaFreeAsync(x, st);
      if (bad & 1) return fail(GTE_CONFIG, "sparse_attention: pattern column out of range");
      return fail(GTE_CONFIG, "sparse_attention: pattern row offsets not monotone");
    }
  }
  if (rows > 0) expand_rows_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(p->row_ptr, rows, row_of_edge);
  iota_kernel<<<grid_for(nnz), 256, 0, st>>>(iota, nnz);
  count_cols_kernel<<<grid_for(nnz), 256, 0, st>>>(p->cols, nnz, counts);
  c->launches += 4;
  int bits = 1;
  while ((1LL << bits) < rows) ++bits;
  size_t tmp_bytes = 0, tmp2 = 0, tmp3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, p->cols, sorted_cols, iota, p->csc_eid, (int)nnz, 0, bits, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, counts, p->col_ptr, (int)(rows + 1), st);
  cub::DeviceReduce::Max(nullptr, tmp3, counts, scratch + 2, (int)rows, st);
  if (tmp2 > tmp_bytes) tmp_bytes = tmp2;
  if (tmp3 > tmp_bytes) tmp_bytes = tmp3;
  void* tmp = nullptr;
  CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes + 16, st));
  if (nnz > 0) CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, p->cols, sorted_cols, iota, p->csc_eid, (int)nnz, 0, bits, st));
  gather_rows_kernel<<<grid_for(nnz), 256, 0, st>>>(p->csc_eid, row_of_edge, nnz, p->csc_row);
  unref_kernel<<<grid_for(rows), 256, 0, st>>>(counts, rows, p->unref, scratch + 1);
  size_t tb = tmp_bytes;
  if (rows > 0) CUDA_TRY(cub::DeviceReduce::Max(tmp, tb, counts, scratch + 2, (int)rows, st));
  tb = tmp_bytes;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, p->col_ptr, (int)(rows + 1), st));
  degree_kernel<<<grid_for(rows), 256, 0, st>>>(p->row_ptr, rows, row_of_edge);  // reuse as row degrees
  tb = tmp_bytes;
  if (rows > 0) CUDA_TRY(cub::DeviceReduce::Max(tmp, tb, row_of_edge, scratch + 3, (int)rows, st));
  c->launches += 8;
  int32_t h[4] = {0, 0, 0, 0};
  CUDA_TRY(cudaMemcpyAsync(h, scratch, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(row_of_edge, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(sorted_cols, st);
  cudaFreeAsync(counts, st);
  cudaFreeAsync(scratch, st);
  p->n_unref = h[1];
  p->max_col_deg = rows > 0 ? h[2] : 0;
  p->max_row_deg = rows > 0 ? h[3] : 0;
  return GTE_OK;
}

// Execution plan of the tile kernels (attn_tile.cuh) for both passes: walk
// the execution order (given, or natural), send rows (columns) longer than
// kHubDegree to the hub list, cut the rest into tiles of <= kTileRows rows
// and <= kTileCap edges, and order each tile longest-first (its slots then
// finish together). An execution order only: outputs do not depend on it.
int build_exec(gte_plan* p, const int64_t* order) {
  const int64_t n = p->rows;
  cudaStream_t st = p->ctx->stream;
  std::vector<int32_t> rp(n + 1), cp(n + 1);
  CUDA_TRY(cudaMemcpyAsync(rp.data(), p->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(cp.data(), p->col_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  struct Pass {
    std::vector<int32_t> order, tiles, hubs;
  } ps[2];
  for (int pass = 0; pass < 2; ++pass) {
    const std::vector<int32_t>& ptr = pass == 0 ? rp : cp;
    Pass& P = ps[pass];
    auto deg = [&](int32_t r) { return ptr[r + 1] - ptr[r]; };
    P.tiles.push_back(0);
    int rows_in = 0, edges_in = 0;
    for (int64_t x = 0; x < n; ++x) {
      const int32_t r = (int32_t)(order ? order[x] : x);
      if (pass == 0 && p->out_rows >= 0 && r >= p->out_rows) continue;  // no outputs wanted (edge-free rows)
      const int dg = deg(r);
      if (dg > kHubDegree) {
        P.hubs.push_back(r);
        continue;
      }
      const int pdg = (dg + 3) / 4 * 4;  // the wide kernels pad rows to 4 edges
      if (rows_in == kTileRows || edges_in + pdg > kTileCap) {
        P.tiles.push_back((int32_t)P.order.size());
        rows_in = edges_in = 0;
      }
      P.order.push_back(r);
      ++rows_in;
      edges_in += pdg;
    }
    if (rows_in > 0) P.tiles.push_back((int32_t)P.order.size());
    for (size_t t = 0; t + 1 < P.tiles.size(); ++t)
      std::stable_sort(P.order.begin() + P.tiles[t], P.order.begin() + P.tiles[t + 1],
                       [&](int32_t a, int32_t b) { return deg(a) > deg(b); });
  }
  size_t total = 0;
  for (auto& P : ps) total += P.order.size() + P.tiles.size() + P.hubs.size();
  cudaFree(p->exec);
  p->exec = nullptr;
  CUDA_TRY(cudaMalloc(&p->exec, sizeof(int32_t) * (total + 1)));
  int32_t* cur = p->exec;
  const int32_t* where[2][3];
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<int32_t>* v[3] = {&ps[pass].order, &ps[pass].tiles, &ps[pass].hubs};
    for (int a = 0; a < 3; ++a) {
      where[pass][a] = cur;
      if (!v[a]->empty())
        CUDA_TRY(cudaMemcpyAsync(cur, v[a]->data(), sizeof(int32_t) * v[a]->size(), cudaMemcpyHostToDevice, st));
      cur += v[a]->size();
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  p->order = where[0][0];
  p->tiles = where[0][1];
  p->hubs = where[0][2];
  p->order_c = where[1][0];
  p->tiles_c = where[1][1];
  p->hubs_c = where[1][2];
  p->n_tiles = (int)ps[0].tiles.size() - 1;
  p->n_hubs = (int)ps[0].hubs.size();
  p->n_tiles_c = (int)ps[1].tiles.size() - 1;
  p->n_hubs_c = (int)ps[1].hubs.size();
  return GTE_OK;
}

void free_plan(gte_plan* p) {
  if (!p) return;
  if (p->ecr) {
    free_plan(p->ecr->rem);
    cudaFree(p->ecr->dev);
    p->ecr->part.release();
    delete p->ecr;
    p->ecr = nullptr;
  }
  cudaFree(p->row_ptr);
  cudaFree(p->cols);
  cudaFree(p->col_ptr);
  cudaFree(p->csc_row);
  cudaFree(p->csc_eid);
  cudaFree(p->unref);
  cudaFree(p->exec);
  delete p;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int pick_dht(int d) { return d <= 8 ? 8 : d <= 16 ? 16 : d <= 32 ? 32 : 64; }
int pick_lpn(int H) {
  int l = 1;
  while (l < H) l <<= 1;
  return l;
}

// Tile family (attn_tile.cuh): f32/bf16, dk == dv, head chunk a
// power-of-two number of 16-byte pieces, all heads of a neighbour within one
// warp, 16-byte aligned rows. Returns lanes-per-head, or 0 if not eligible.
int fast_lph(int dtype, int64_t S, int H, int dk, int dv, int64_t ldq, int64_t ldv,
             std::initializer_list<const void*> ptrs) {
  // 32-bit gather offsets inside the kernels
  if ((S + 1) * (ldq > ldv ? ldq : ldv) * (int64_t)elem_size(dtype) >= (int64_t(1) << 32)) return 0;
  if (dtype != GTE_F32 && dtype != GTE_BF16) return 0;
  if (dk != dv) return 0;
  const int64_t es = (int64_t)elem_size(dtype);
  if ((dk * es) % 16 != 0 || (ldq * es) % 16 != 0 || (ldv * es) % 16 != 0) return 0;
  const int lph = (int)(dk * es / 16);
  if (lph != 1 && lph != 2 && lph != 4 && lph != 8) return 0;
  int lpn = 1;
  while (lpn < H) lpn <<= 1;
  if (lpn * lph > 32) return 0;
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return 0;
  return lph;
}

}  // namespace
namespace {

cudaError_t dispatch_tile(int dtype, int which, const SparseArgs& a, int lph, cudaStream_t st, int64_t* launches) {
  int lpn = 1;
  while (lpn < a.H) lpn <<= 1;
  lpn *= lph;
  int n = 0;
  cudaError_t e = dtype == GTE_F32 ? launch_tile_f32(which, a, lph, lpn, st, &n)
                                   : launch_tile_bf16(which, a, lph, lpn, st, &n);
  *launches += n;
  return e;
}

cudaError_t dispatch(int dtype, int which, const SparseArgs& a, int dht, int lpn, cudaStream_t st) {
  switch (dtype) {
    case GTE_F64: return launch_sparse_f64(which, a, dht, lpn, st);
    case GTE_F32: return launch_sparse_f32(which, a, dht, lpn, st);
    default: return launch_sparse_bf16(which, a, dht, lpn, st);
  }
}

int check_attn_args(const gte_plan* plan, int dtype, int H, int dk, int dv, int64_t ldq, int64_t ldv) {
  if (!plan) return fail(GTE_CONFIG, "sparse_attention: null plan");
  if (dtype != GTE_F64 && dtype != GTE_F32 && dtype != GTE_BF16) return fail(GTE_CONFIG, "sparse_attention: bad dtype");
  if (dk < 1) return fail(GTE_CONFIG, "attention: d_K must be >= 1");
  if (dv < 1) return fail(GTE_CONFIG, "attention: d_V must be >= 1");
  if (dk > 64 || dv > 64) return fail(GTE_CONFIG, "sparse_attention: head dim > 64 unsupported");
  if (H < 1 || H > 32) return fail(GTE_CONFIG, "sparse_attention: heads must lie in [1, 32]");
  if (ldq < (int64_t)H * dk || ldv < (int64_t)H * dv) return fail(GTE_CONFIG, "sparse_attention: leading dimension too small");
  return GTE_OK;
}

void fill_common(SparseArgs& a, const gte_plan* plan, int dtype, int H, int dk, int dv, int64_t ldq, int64_t ldv) {
  a.S = plan->rows;
  a.E = plan->nnz;
  a.H = H;
  a.dk = dk;
  a.dv = dv;
  a.ldq = ldq;
  a.ldv = ldv;
  a.row_ptr = plan->row_ptr;
  a.cols = plan->cols;
  a.col_ptr = plan->col_ptr;
  a.csc_row = plan->csc_row;
  a.csc_eid = plan->csc_eid;
  a.scale = 1.0 / std::sqrt((double)dk);
  a.scale_l = (float)a.scale * 1.4426950408889634f;  // == the kernels' former float(scale) * kLogScale
  a.rq_bytes = (uint32_t)(ldq * (int64_t)elem_size(dtype));
  a.rv_bytes = (uint32_t)(ldv * (int64_t)elem_size(dtype));
  a.err = plan->ctx->d_err;
  a.order = plan->order;
  a.tiles = plan->tiles;
  a.hubs = plan->hubs;
  a.order_c = plan->order_c;
  a.tiles_c = plan->tiles_c;
  a.hubs_c = plan->hubs_c;
  a.n_tiles = plan->n_tiles;
  a.n_hubs = plan->n_hubs;
  a.n_tiles_c = plan->n_tiles_c;
  a.n_hubs_c = plan->n_hubs_c;
  (void)dtype;
}

}  // namespace

extern "C" {

const char* gte_last_error(void) { return g_err.c_str(); }
const char* gte_version(void) { return "gte_b200 0.1 (sm_100a)"; }

int gte_ctx_create(int device, gte_ctx** out) {
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new gte_ctx();
  c->device = device;
  c->stream = nullptr;  // legacy default stream until set
  CUDA_TRY(cudaMalloc(&c->d_err, 2 * sizeof(int)));
  CUDA_TRY(cudaMallocHost(&c->h_err, 2 * sizeof(int)));
  int rc = reset_err(c);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *out = c;
  return GTE_OK;
}

int gte_ctx_destroy(gte_ctx* c) {
  if (!c) return GTE_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamSynchronize(c->down);
    cudaStreamDestroy(c->copy);
    cudaStreamDestroy(c->down);
    for (auto& e : c->ev) cudaEventDestroy(e);
    for (int s = 0; s < 2; ++s) {
      cudaEventDestroy(c->k_done[s]);
      cudaEventDestroy(c->d2h_done[s]);
      for (auto& b : c->hs[s]) b.release();
    }
  }
  for (auto& b : c->io) b.release();
  c->scratch.release();
  cudaFree(c->d_err);
  cudaFreeHost(c->h_err);
  delete c;
  return GTE_OK;
}

// device memory for C/C++ callers without the CUDA runtime (the drop-in bridge)
int gte_dev_alloc(gte_ctx* c, int64_t bytes, void** out) {
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMalloc(out, bytes > 0 ? (size_t)bytes : 16));
  return GTE_OK;
}
int gte_dev_free(gte_ctx* c, void* p) {
  if (p) {
    cudaStreamSynchronize(c->stream);
    cudaFree(p);
  }
  return GTE_OK;
}
int gte_copy_h2d(gte_ctx* c, void* dst, const void* src, int64_t bytes) {
  if (bytes > 0) CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, c->stream));
  return GTE_OK;
}
int gte_copy_d2h(gte_ctx* c, void* dst, const void* src, int64_t bytes) {
  if (bytes > 0) CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return GTE_OK;
}

int gte_ctx_set_stream(gte_ctx* c, void* s) {
  c->stream = static_cast<cudaStream_t>(s);
  return GTE_OK;
}

int gte_ctx_sync(gte_ctx* c) {
  if (c->down) {  // in-flight asynchronous fwd_bwd_host steps
    CUDA_TRY(cudaStreamSynchronize(c->down));
    c->pending = false;
  }
  return drain_errors(c);
}

int64_t gte_ctx_launches(const gte_ctx* c) { return c->launches; }

int gte_plan_create_device(gte_ctx* c, int64_t rows, int64_t nnz, const int32_t* d_row_ptr,
                           const int32_t* d_cols, gte_plan** out) {
  if (rows < 0 || nnz < 0) return fail(GTE_CONFIG, "plan: negative size");
  if (rows >= INT_MAX || nnz >= INT_MAX) return fail(GTE_CONFIG, "plan: pattern exceeds int32 device index range");
  auto* p = new gte_plan();
  p->ctx = c;
  p->rows = rows;
  p->nnz = nnz;
  cudaStream_t st = c->stream;
  if (cudaMallocAsync(&p->row_ptr, sizeof(int32_t) * (rows + 1), st) != cudaSuccess ||
      cudaMallocAsync(&p->cols, sizeof(int32_t) * (nnz + 1), st) != cudaSuccess) {
    free_plan(p);
    return fail(GTE_CUDA, "plan: device allocation failed");
  }
  cudaMemcpyAsync(p->row_ptr, d_row_ptr, sizeof(int32_t) * (rows + 1), cudaMemcpyDeviceToDevice, st);
  if (nnz) cudaMemcpyAsync(p->cols, d_cols, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, st);
  int rc = build_plan_device(c, p);
  if (rc == GTE_OK) rc = build_exec(p, nullptr);
  if (rc) {
    free_plan(p);
    return rc;
  }
  *out = p;
  return GTE_OK;
}

int gte_plan_create_host(gte_ctx* c, int64_t rows, int64_t nnz, const int64_t* row_off,
                         const int64_t* cols, gte_plan** out) {
  if (rows < 0 || nnz < 0) return fail(GTE_CONFIG, "plan: negative size");
  if (rows >= INT_MAX || nnz >= INT_MAX) return fail(GTE_CONFIG, "plan: pattern exceeds int32 device index range");
  if (row_off[0] != 0 || row_off[rows] != nnz) return fail(GTE_CONFIG, "sparse_attention: malformed pattern offsets");
  // host-side validation before narrowing to the int32 device indices: a
  // column >= 2^31 must not wrap into a valid id
  std::vector<int32_t> ro(rows + 1), co(nnz > 0 ? nnz : 1);
  for (int64_t i = 0; i < rows; ++i)
    if (row_off[i + 1] < row_off[i]) return fail(GTE_CONFIG, "sparse_attention: pattern row offsets not monotone");
  for (int64_t i = 0; i <= rows; ++i) ro[i] = (int32_t)row_off[i];
  for (int64_t i = 0; i < nnz; ++i) {
    if (cols[i] < 0 || cols[i] >= rows) return fail(GTE_CONFIG, "sparse_attention: pattern column out of range");
    co[i] = (int32_t)cols[i];
  }
  auto* p = new gte_plan();
  p->ctx = c;
  p->rows = rows;
  p->nnz = nnz;
  cudaStream_t st = c->stream;
  if (cudaMalloc(&p->row_ptr, sizeof(int32_t) * (rows + 1)) != cudaSuccess ||
      cudaMalloc(&p->cols, sizeof(int32_t) * (nnz + 1)) != cudaSuccess) {
    free_plan(p);
    return fail(GTE_CUDA, "plan: device allocation failed");
  }
  cudaMemcpyAsync(p->row_ptr, ro.data(), sizeof(int32_t) * (rows + 1), cudaMemcpyHostToDevice, st);
  if (nnz) cudaMemcpyAsync(p->cols, co.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
  int rc = build_plan_device(c, p);  // synchronises before `ro`/`co` go out of scope
  if (rc == GTE_OK) rc = build_exec(p, nullptr);
  if (rc) {
    free_plan(p);
    return rc;
  }
  *out = p;
  return GTE_OK;
}

int gte_plan_destroy(gte_plan* p) {
  if (p) cudaStreamSynchronize(p->ctx->stream);
  free_plan(p);
  return GTE_OK;
}

int gte_plan_shape(const gte_plan* p, int64_t* rows, int64_t* nnz, int64_t* mr, int64_t* mc) {
  if (rows) *rows = p->rows;
  if (nnz) *nnz = p->nnz;
  if (mr) *mr = p->max_row_deg;
  if (mc) *mc = p->max_col_deg;
  return GTE_OK;
}

int gte_plan_device_csr(const gte_plan* p, const int32_t** rp, const int32_t** cl) {
  *rp = p->row_ptr;
  *cl = p->cols;
  return GTE_OK;
}

int gte_plan_set_order(gte_plan* p, const int64_t* order) {
  if (!p) return fail(GTE_CONFIG, "plan: null plan");
  const int64_t n = p->rows;
  if (order) {
    std::vector<char> seen(n > 0 ? n : 1, 0);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t r = order[i];
      if (r < 0 || r >= n || seen[r]) return fail(GTE_CONFIG, "plan: order is not a permutation of the rows");
      seen[r] = 1;
    }
  }
  int rc = build_exec(p, order);
  if (rc) return rc;
  p->scheduled = order != nullptr;
  if (!order) p->communities = 0;
  if (order) p->host_order.assign(order, order + n);
  else p->host_order.clear();
  if (p->ecr && p->ecr->rem) return gte_plan_set_order(p->ecr->rem, order);
  return GTE_OK;
}

// Rows [n, rows) produce no outputs: the forward and the backward's CSR pass
// skip them (their O / LSE / dQ rows are left unwritten); they must have no
// edges. The CSC pass still covers every column. For a sequence-parallel
// rank's local plan, whose trailing halo rows only exist as columns.
int gte_plan_set_output_rows(gte_plan* p, int64_t n) {
  if (!p) return fail(GTE_CONFIG, "plan: null plan");
  if (n < 0 || n > p->rows) return fail(GTE_CONFIG, "plan: output rows out of range");
  int32_t off = 0;
  CUDA_TRY(cudaMemcpy(&off, p->row_ptr + n, sizeof off, cudaMemcpyDeviceToHost));
  if (off != p->nnz) return fail(GTE_CONFIG, "plan: rows without outputs must have no edges");
  p->out_rows = n == p->rows ? -1 : n;
  int rc = build_exec(p, p->host_order.empty() ? nullptr : p->host_order.data());
  if (rc) return rc;
  if (p->ecr && p->ecr->rem) return gte_plan_set_output_rows(p->ecr->rem, n);
  return GTE_OK;
}

// Registers the ECR sub-blocks of a cluster-sparse layout (global origins
// (row0, col0), side d_b): their pairs run as dense tiles on the tensor pipe
// (bf16, ecr_tile.cuh), the rest of the pattern on the sparse kernels. Every
// sub-block must lie in the pattern as 16 contiguous column runs and no pair
// may belong to two sub-blocks (the layout guarantees both:
// reformation.cpp:82-99, 176-189). Sub-blocks touching a row or column of
// degree > kHubDegree stay on the sparse path (hub kernels), and d_b != 16
// registers nothing. Results do not depend on the split beyond rounding.
int gte_plan_set_blocks(gte_plan* p, int64_t n_blocks, const int64_t* origins, int64_t d_b, int64_t* n_used) {
  if (!p) return fail(GTE_CONFIG, "plan: null plan");
  if (n_used) *n_used = 0;
  if (p->ecr) {
    free_plan(p->ecr->rem);
    cudaFree(p->ecr->dev);
    p->ecr->part.release();
    delete p->ecr;
    p->ecr = nullptr;
  }
  if (n_blocks < 0) return fail(GTE_CONFIG, "blocks: negative count");
  if (n_blocks == 0 || d_b != kEcrDb) return GTE_OK;
  const int64_t n = p->rows, m = p->nnz;
  cudaStream_t st = p->ctx->stream;
  std::vector<int32_t> rp(n + 1), cl(m > 0 ? m : 1), cp(n + 1);
  CUDA_TRY(cudaMemcpyAsync(rp.data(), p->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(cp.data(), p->col_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (m) CUDA_TRY(cudaMemcpyAsync(cl.data(), p->cols, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<char> taken(m > 0 ? m : 1, 0);
  std::vector<int32_t> blk, ebase;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const int64_t r0 = origins[2 * b], c0 = origins[2 * b + 1];
    if (r0 < 0 || c0 < 0 || r0 + d_b > n || c0 + d_b > n)
      return fail(GTE_CONFIG, "blocks: sub-block outside the sequence");
    bool hub = false;
    for (int64_t t = 0; t < d_b; ++t)
      hub |= rp[r0 + t + 1] - rp[r0 + t] > kHubDegree || cp[c0 + t + 1] - cp[c0 + t] > kHubDegree;
    int32_t eb[kEcrDb];
    for (int64_t t = 0; t < d_b; ++t) {
      const int32_t* b0 = cl.data() + rp[r0 + t];
      const int32_t* b1 = cl.data() + rp[r0 + t + 1];
      const int32_t* at = std::lower_bound(b0, b1, (int32_t)c0);
      if (b1 - at < d_b || at[d_b - 1] != (int32_t)(c0 + d_b - 1))
        return fail(GTE_CONFIG, "blocks: sub-block (" + std::to_string(r0) + ", " + std::to_string(c0) +
                                    ") is not inside the pattern");
      eb[t] = (int32_t)(at - cl.data());
    }
    if (hub) continue;
    for (int64_t t = 0; t < d_b; ++t)
      for (int64_t u = 0; u < d_b; ++u) {
        if (taken[eb[t] + u]) return fail(GTE_CONFIG, "blocks: sub-blocks overlap");
        taken[eb[t] + u] = 1;
      }
    blk.push_back((int32_t)r0);
    blk.push_back((int32_t)c0);
    ebase.insert(ebase.end(), eb, eb + d_b);
  }
  const int64_t nb = (int64_t)blk.size() / 2;
  if (nb == 0) return GTE_OK;
  // incidences: per row (column) the sub-blocks covering it, in block order
  std::vector<int32_t> inc_ptr(n + 1, 0), cinc_ptr(n + 1, 0), inc(nb * d_b), cinc(nb * d_b);
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t t = 0; t < d_b; ++t) {
      inc_ptr[blk[2 * b] + t + 1]++;
      cinc_ptr[blk[2 * b + 1] + t + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) {
    inc_ptr[i + 1] += inc_ptr[i];
    cinc_ptr[i + 1] += cinc_ptr[i];
  }
  {
    std::vector<int32_t> fr(inc_ptr.begin(), inc_ptr.end() - 1), fc(cinc_ptr.begin(), cinc_ptr.end() - 1);
    for (int64_t b = 0; b < nb; ++b)
      for (int64_t t = 0; t < d_b; ++t) {
        inc[b * d_b + t] = fr[blk[2 * b] + t]++;
        cinc[b * d_b + t] = fc[blk[2 * b + 1] + t]++;
      }
  }
  // remainder pattern (CSR positions -> original edge ids)
  std::vector<int64_t> rro(n + 1, 0), rco;
  std::vector<int32_t> eid;
  rco.reserve(m);
  eid.reserve(m);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (!taken[e]) {
        rco.push_back(cl[e]);
        eid.push_back((int32_t)e);
      }
    rro[i + 1] = (int64_t)rco.size();
  }
  auto* x = new EcrSplit();
  x->n_blocks = nb;
  x->n_inc = inc_ptr[n];
  x->n_cinc = cinc_ptr[n];
  const int64_t mr = (int64_t)rco.size();
  int rc = gte_plan_create_host(p->ctx, n, mr, rro.data(), mr ? rco.data() : rro.data(), &x->rem);
  if (rc) {
    delete x;
    return rc;
  }
  p->ecr = x;
  if (!p->host_order.empty()) {
    rc = gte_plan_set_order(x->rem, p->host_order.data());
    if (rc) return rc;
  }
  // the remainder's CSC edge ids -> original edge ids
  if (mr) {
    std::vector<int32_t> ce(mr);
    CUDA_TRY(cudaMemcpyAsync(ce.data(), x->rem->csc_eid, sizeof(int32_t) * mr, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (auto& v : ce) v = eid[v];
    CUDA_TRY(cudaMemcpyAsync(x->rem->csc_eid, ce.data(), sizeof(int32_t) * mr, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  const size_t total = blk.size() + ebase.size() + inc.size() + cinc.size() + 2 * (n + 1) + eid.size() + 1;
  CUDA_TRY(cudaMalloc(&x->dev, sizeof(int32_t) * total));
  int32_t* cur = x->dev;
  auto put = [&](const std::vector<int32_t>& v, const int32_t** where) -> cudaError_t {
    *where = cur;
    cudaError_t e = v.empty() ? cudaSuccess
                              : cudaMemcpyAsync(cur, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, st);
    cur += v.size();
    return e;
  };
  CUDA_TRY(put(blk, &x->blk));
  CUDA_TRY(put(ebase, &x->ebase));
  CUDA_TRY(put(inc, &x->inc));
  CUDA_TRY(put(cinc, &x->cinc));
  CUDA_TRY(put(inc_ptr, &x->inc_ptr));
  CUDA_TRY(put(cinc_ptr, &x->cinc_ptr));
  CUDA_TRY(put(eid, &x->eid));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (n_used) *n_used = nb;
  return GTE_OK;
}

int gte_plan_blocks(const gte_plan* p, int64_t* n_blocks, int64_t* remainder_nnz) {
  if (!p) return fail(GTE_CONFIG, "plan: null plan");
  if (n_blocks) *n_blocks = p->ecr ? p->ecr->n_blocks : 0;
  if (remainder_nnz) *remainder_nnz = p->ecr ? p->ecr->rem->nnz : p->nnz;
  return GTE_OK;
}

int gte_plan_schedule(gte_plan* p, int64_t iters, int64_t* communities) {
  if (!p) return fail(GTE_CONFIG, "plan: null plan");
  const int64_t n = p->rows, m = p->nnz;
  cudaStream_t st = p->ctx->stream;
  std::vector<int32_t> ro(n + 1), co(m > 0 ? m : 1);
  CUDA_TRY(cudaMemcpyAsync(ro.data(), p->row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (m) CUDA_TRY(cudaMemcpyAsync(co.data(), p->cols, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int64_t> ro64(ro.begin(), ro.end()), co64(co.begin(), co.begin() + m), order(n > 0 ? n : 1);
  int64_t comms = 0;
  int rc = gte_community_order(n, m, ro64.data(), co64.data(), iters, order.data(), &comms);
  if (rc) return rc;
  rc = gte_plan_set_order(p, order.data());
  if (rc) return rc;
  p->communities = comms;
  if (communities) *communities = comms;
  return GTE_OK;
}

namespace {

// The ECR split runs when sub-blocks are registered, the tile path is taken,
// the dtype is bf16 (tensor-core tiles) and the head geometry has kernels.
EcrSplit* ecr_split_for(const gte_plan* plan, int dtype, int lph, int H, int dk, int dv) {
  EcrSplit* x = plan->ecr;
  if (!x || x->n_blocks == 0 || !lph || dtype != GTE_BF16 || !ecr_eligible(H, dk, dv)) return nullptr;
  return x;
}

cudaError_t ecr_prepare(EcrSplit* x, const gte_plan* plan, int H, int dk, int64_t ldq, int64_t ldv, EcrArgs& e,
                        SparseArgs& a2, float** part) {
  const size_t D = (size_t)H * dk;
  const size_t fwd = (size_t)x->n_inc * (2 * H + D), bwd = (size_t)x->n_inc * D + 2 * (size_t)x->n_cinc * D;
  cudaError_t err = x->part.ensure(sizeof(float) * (fwd > bwd ? fwd : bwd));
  if (err != cudaSuccess) return err;
  *part = static_cast<float*>(x->part.p);
  e.n_blocks = (int)x->n_blocks;
  e.H = H;
  e.dh = dk;
  e.E = plan->nnz;
  e.ldq = ldq;
  e.ldv = ldv;
  e.scale = (float)(1.0 / std::sqrt((double)dk));
  e.blk = x->blk;
  e.ebase = x->ebase;
  e.inc = x->inc;
  e.cinc = x->cinc;
  a2.E = plan->nnz;  // weight_mult rows stay [H][E] of the full pattern
  a2.eid = x->eid;
  a2.inc_ptr = x->inc_ptr;
  a2.part_d = (int)D;
  return cudaSuccess;
}

}  // namespace

int gte_sparse_attn_fwd(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                        const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                        const void* bias, const void* wmult, void* out, void* lse, int flags) {
  int rc = check_attn_args(plan, dtype, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  SparseArgs a;
  fill_common(a, plan, dtype, H, dk, dv, ldq, ldv);
  a.q = q;
  a.k = k;
  a.v = v;
  a.bias = bias;
  a.wmult = wmult;
  a.out = out;
  a.lse = lse;
  a.forbid_empty = (flags & GTE_FORBID_EMPTY_ROWS) ? 1 : 0;
  const int dht = pick_dht(dk > dv ? dk : dv), lpn = pick_lpn(H);
  const size_t es = elem_size(dtype);
  a.vec_qk = dk == dht && (ldq * es) % 16 == 0 && aligned16(q) && aligned16(k);
  a.vec_v = dv == dht && (ldv * es) % 16 == 0 && aligned16(v) && aligned16(out);
  if (plan->rows == 0) return GTE_OK;
  const int lph = fast_lph(dtype, plan->rows, H, dk, dv, ldq, ldv, {q, k, v, out});
  if (EcrSplit* x = ecr_split_for(plan, dtype, lph, H, dk, dv)) {
    // ECR: dense sub-blocks on the tensor pipe, then the remainder folds their partials in
    EcrArgs e;
    SparseArgs a2 = a;
    fill_common(a2, x->rem, dtype, H, dk, dv, ldq, ldv);
    float* part = nullptr;
    CUDA_TRY(ecr_prepare(x, plan, H, dk, ldq, ldv, e, a2, &part));
    e.q = q;
    e.k = k;
    e.v = v;
    e.bias = static_cast<const float*>(bias);
    e.wmult = static_cast<const float*>(wmult);
    e.part_ml = reinterpret_cast<float2*>(part);
    e.part_acc = part + 2 * (size_t)H * x->n_inc;
    CUDA_TRY(launch_ecr_bf16(false, e, c->stream));
    c->launches += 1;
    a2.part_ml = e.part_ml;
    a2.part_acc = e.part_acc;
    CUDA_TRY(dispatch_tile(dtype, kFwd, a2, lph, c->stream, &c->launches));
  } else if (lph) {
    CUDA_TRY(dispatch_tile(dtype, kFwd, a, lph, c->stream, &c->launches));
  } else {
    CUDA_TRY(dispatch(dtype, kFwd, a, dht, lpn, c->stream));
    c->launches += 1;
  }
  if (!lph && plan->n_unref > 0) {  // the fast kernels check every row's own K/V
    CUDA_TRY(launch_finite_rows(dtype, k, v, plan->unref, (int)plan->n_unref, ldq, ldv, (int64_t)H * dk,
                                (int64_t)H * dv, c->d_err, c->stream));
    c->launches += 1;
  }
  return GTE_OK;
}

int gte_sparse_attn_bwd(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                        const void* q, const void* k, int64_t ldq, const void* v, int64_t ldv,
                        const void* out, const void* lse, const void* dout, const void* bias,
                        const void* wmult, void* dq, void* dk_out, void* dv_out, void* dbias) {
  int rc = check_attn_args(plan, dtype, H, dk, dv, ldq, ldv);
  if (rc) return rc;
  if (plan->rows == 0) return GTE_OK;
  DevBuf& ws = c->io[11];
  CUDA_TRY(ws.ensure(acc_size(dtype) * (size_t)plan->rows * H));
  DevBuf& ws2 = c->io[12];
  CUDA_TRY(ws2.ensure(2 * sizeof(float) * (size_t)plan->rows * H));
  SparseArgs a;
  fill_common(a, plan, dtype, H, dk, dv, ldq, ldv);
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = out;
  a.dout = dout;
  a.bias = bias;
  a.wmult = wmult;
  a.lse = const_cast<void*>(lse);
  a.delta = ws.p;
  a.lsedelta = ws2.p;
  a.dq = dq;
  a.dk_out = dk_out;
  a.dv_out = dv_out;
  a.dbias = dbias;
  const int dht = pick_dht(dk > dv ? dk : dv), lpn = pick_lpn(H);
  const size_t es = elem_size(dtype);
  a.vec_qk = dk == dht && (ldq * es) % 16 == 0 && aligned16(q) && aligned16(k) && aligned16(dq) && aligned16(dk_out);
  a.vec_v = dv == dht && (ldv * es) % 16 == 0 && aligned16(v) && aligned16(out) && aligned16(dout) && aligned16(dv_out);
  const int lph = fast_lph(dtype, plan->rows, H, dk, dv, ldq, ldv, {q, k, v, out, dout, dq, dk_out, dv_out});
  if (EcrSplit* x = ecr_split_for(plan, dtype, lph, H, dk, dv)) {
    // ECR: sub-block partials (dQ rows, dK/dV columns, final dbias of their
    // pairs) first, then the remainder's two passes add them in
    EcrArgs e;
    SparseArgs a2 = a;
    fill_common(a2, x->rem, dtype, H, dk, dv, ldq, ldv);
    float* part = nullptr;
    CUDA_TRY(ecr_prepare(x, plan, H, dk, ldq, ldv, e, a2, &part));
    const size_t D = (size_t)H * dk;
    e.q = q;
    e.k = k;
    e.v = v;
    e.o = out;
    e.dout = dout;
    e.bias = static_cast<const float*>(bias);
    e.wmult = static_cast<const float*>(wmult);
    e.lse = static_cast<const float*>(lse);
    e.part_acc = part;
    e.part_dk = part + D * x->n_inc;
    e.part_dv = e.part_dk + D * x->n_cinc;
    e.dbias = static_cast<float*>(dbias);
    CUDA_TRY(launch_ecr_bf16(true, e, c->stream));
    c->launches += 1;
    a2.cinc_ptr = x->cinc_ptr;
    a2.part_acc = e.part_acc;
    a2.part_dk = e.part_dk;
    a2.part_dv = e.part_dv;
    CUDA_TRY(dispatch_tile(dtype, kBwdRows, a2, lph, c->stream, &c->launches));
    CUDA_TRY(dispatch_tile(dtype, kBwdCols, a2, lph, c->stream, &c->launches));
  } else if (lph) {
    CUDA_TRY(dispatch_tile(dtype, kBwdRows, a, lph, c->stream, &c->launches));
    CUDA_TRY(dispatch_tile(dtype, kBwdCols, a, lph, c->stream, &c->launches));
  } else {
    CUDA_TRY(dispatch(dtype, kBwdRows, a, dht, lpn, c->stream));
    CUDA_TRY(dispatch(dtype, kBwdCols, a, dht, lpn, c->stream));
    c->launches += 2;
  }
  return GTE_OK;
}

int gte_sparse_attn_fwd_host(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                             const void* q, const void* k, const void* v, const void* bias,
                             const void* wmult, void* out, void* lse_out, int flags) {
  int rc = check_attn_args(plan, dtype, H, dk, dv, (int64_t)H * dk, (int64_t)H * dv);
  if (rc) return rc;
  const size_t S = (size_t)plan->rows, E = (size_t)plan->nnz, es = elem_size(dtype), as = acc_size(dtype);
  const size_t bq = S * H * dk * es, bv = S * H * dv * es;
  cudaStream_t st = c->stream;
  CUDA_TRY(c->io[0].ensure(bq));
  CUDA_TRY(c->io[1].ensure(bq));
  CUDA_TRY(c->io[2].ensure(bv));
  CUDA_TRY(c->io[3].ensure(bv));
  CUDA_TRY(c->io[4].ensure(S * H * as));
  if (bias) CUDA_TRY(c->io[5].ensure(E * as));
  if (wmult) CUDA_TRY(c->io[6].ensure(E * H * as));
  CUDA_TRY(cudaMemcpyAsync(c->io[0].p, q, bq, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[1].p, k, bq, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[2].p, v, bv, cudaMemcpyHostToDevice, st));
  if (bias) CUDA_TRY(cudaMemcpyAsync(c->io[5].p, bias, E * as, cudaMemcpyHostToDevice, st));
  if (wmult) CUDA_TRY(cudaMemcpyAsync(c->io[6].p, wmult, E * H * as, cudaMemcpyHostToDevice, st));
  rc = gte_sparse_attn_fwd(c, plan, dtype, H, dk, dv, c->io[0].p, c->io[1].p, (int64_t)H * dk, c->io[2].p,
                           (int64_t)H * dv, bias ? c->io[5].p : nullptr, wmult ? c->io[6].p : nullptr,
                           c->io[3].p, c->io[4].p, flags);
  if (rc) return rc;
  rc = drain_errors(c, (flags & GTE_IGNORE_NONFINITE) != 0);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, c->io[3].p, bv, cudaMemcpyDeviceToHost, st));
  if (lse_out) CUDA_TRY(cudaMemcpyAsync(lse_out, c->io[4].p, S * H * as, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return GTE_OK;
}

int gte_sparse_attn_bwd_host(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                             const void* q, const void* k, const void* v, const void* out,
                             const void* lse, const void* dout, const void* bias,
                             const void* wmult, void* dq, void* dk_out, void* dv_out, void* dbias) {
  int rc = check_attn_args(plan, dtype, H, dk, dv, (int64_t)H * dk, (int64_t)H * dv);
  if (rc) return rc;
  const size_t S = (size_t)plan->rows, E = (size_t)plan->nnz, es = elem_size(dtype), as = acc_size(dtype);
  const size_t bq = S * H * dk * es, bv = S * H * dv * es;
  cudaStream_t st = c->stream;
  for (int i : {0, 1, 7, 8}) CUDA_TRY(c->io[i].ensure(bq));
  for (int i : {2, 3, 9, 10}) CUDA_TRY(c->io[i].ensure(bv));
  CUDA_TRY(c->io[4].ensure(S * H * as));
  CUDA_TRY(c->io[5].ensure((E + 1) * as));
  if (wmult) CUDA_TRY(c->io[6].ensure(E * H * as));
  CUDA_TRY(cudaMemcpyAsync(c->io[0].p, q, bq, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[1].p, k, bq, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[2].p, v, bv, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[3].p, out, bv, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[4].p, lse, S * H * as, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->io[9].p, dout, bv, cudaMemcpyHostToDevice, st));
  void* dbias_dev = c->io[5].p;
  DevBuf bias_buf;
  const void* bias_dev = nullptr;
  if (bias) {
    CUDA_TRY(bias_buf.ensure(E * as));
    CUDA_TRY(cudaMemcpyAsync(bias_buf.p, bias, E * as, cudaMemcpyHostToDevice, st));
    bias_dev = bias_buf.p;
  }
  if (wmult) CUDA_TRY(cudaMemcpyAsync(c->io[6].p, wmult, E * H * as, cudaMemcpyHostToDevice, st));
  rc = gte_sparse_attn_bwd(c, plan, dtype, H, dk, dv, c->io[0].p, c->io[1].p, (int64_t)H * dk, c->io[2].p,
                           (int64_t)H * dv, c->io[3].p, c->io[4].p, c->io[9].p, bias_dev,
                           wmult ? c->io[6].p : nullptr, c->io[7].p, c->io[8].p, c->io[10].p, dbias_dev);
  if (rc == GTE_OK) {
    CUDA_TRY(cudaMemcpyAsync(dq, c->io[7].p, bq, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(dk_out, c->io[8].p, bq, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(dv_out, c->io[10].p, bv, cudaMemcpyDeviceToHost, st));
    if (dbias && E) CUDA_TRY(cudaMemcpyAsync(dbias, dbias_dev, E * as, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  bias_buf.release();
  return rc;
}

// One fwd+bwd unit with host buffers. Three streams: uploads (c->copy),
// kernels (c->stream), downloads (c->down), ordered by events; dO travels
// while the forward runs, O comes back while the backward runs. The async
// variant returns after enqueueing: the next step's uploads then overlap this
// step's downloads (each engine direction busy at once); gte_ctx_sync waits.
static int fwd_bwd_host_impl(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv, const void* q,
                             const void* k, const void* v, const void* dout, const void* bias, void* out, void* dq,
                             void* dk_out, void* dv_out, void* dbias, bool sync) {
  int rc = check_attn_args(plan, dtype, H, dk, dv, (int64_t)H * dk, (int64_t)H * dv);
  if (rc) return rc;
  const size_t S = (size_t)plan->rows, E = (size_t)plan->nnz, es = elem_size(dtype), as = acc_size(dtype);
  const size_t bq = S * H * dk * es, bv = S * H * dv * es;
  cudaStream_t st = c->stream;
  if (!c->copy) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking));
    for (auto& e : c->ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int s = 0; s < 2; ++s) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->k_done[s], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->d2h_done[s], cudaEventDisableTiming));
    }
  }
  const int sidx = c->parity;
  c->parity ^= 1;
  DevBuf* B = c->hs[sidx];
  const bool grow = B[0].cap < bq || B[2].cap < bv || B[4].cap < S * H * as || B[5].cap < (E + 1) * as ||
                    B[6].cap < (E + 1) * as;
  if (grow && c->pending) {  // this set's buffers are about to move: finish what is in flight
    CUDA_TRY(cudaStreamSynchronize(c->down));
    CUDA_TRY(cudaStreamSynchronize(st));
    c->pending = false;
  }
  for (int i : {0, 1, 7, 8}) CUDA_TRY(B[i].ensure(bq));
  for (int i : {2, 3, 9, 10}) CUDA_TRY(B[i].ensure(bv));
  CUDA_TRY(B[4].ensure(S * H * as));
  CUDA_TRY(B[5].ensure((E + 1) * as));
  CUDA_TRY(B[6].ensure((E + 1) * as));
  cudaStream_t up = c->copy, dn = c->down;
  const bool used = c->hs_used[sidx] && !grow;
  c->hs_used[sidx] = true;
  // uploads into this set wait for the kernels of the step that last used it
  if (used) CUDA_TRY(cudaStreamWaitEvent(up, c->k_done[sidx], 0));
  CUDA_TRY(cudaMemcpyAsync(B[1].p, k, bq, cudaMemcpyHostToDevice, up));
  CUDA_TRY(cudaMemcpyAsync(B[2].p, v, bv, cudaMemcpyHostToDevice, up));
  CUDA_TRY(cudaMemcpyAsync(B[0].p, q, bq, cudaMemcpyHostToDevice, up));
  if (bias) CUDA_TRY(cudaMemcpyAsync(B[6].p, bias, E * as, cudaMemcpyHostToDevice, up));
  CUDA_TRY(cudaEventRecord(c->ev[0], up));  // forward inputs resident
  CUDA_TRY(cudaMemcpyAsync(B[9].p, dout, bv, cudaMemcpyHostToDevice, up));
  CUDA_TRY(cudaEventRecord(c->ev[1], up));  // dO resident
  const void* bias_dev = bias ? B[6].p : nullptr;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev[0], 0));
  // outputs of this set are free once their previous download finished
  if (used) CUDA_TRY(cudaStreamWaitEvent(st, c->d2h_done[sidx], 0));
  rc = gte_sparse_attn_fwd(c, plan, dtype, H, dk, dv, B[0].p, B[1].p, (int64_t)H * dk, B[2].p, (int64_t)H * dv,
                           bias_dev, nullptr, B[3].p, B[4].p, 0);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->ev[2], st));  // O ready
  CUDA_TRY(cudaStreamWaitEvent(dn, c->ev[2], 0));
  CUDA_TRY(cudaMemcpyAsync(out, B[3].p, bv, cudaMemcpyDeviceToHost, dn));
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev[1], 0));
  rc = gte_sparse_attn_bwd(c, plan, dtype, H, dk, dv, B[0].p, B[1].p, (int64_t)H * dk, B[2].p, (int64_t)H * dv,
                           B[3].p, B[4].p, B[9].p, bias_dev, nullptr, B[7].p, B[8].p, B[10].p, B[5].p);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(c->k_done[sidx], st));  // gradients ready; this set's inputs free
  CUDA_TRY(cudaStreamWaitEvent(dn, c->k_done[sidx], 0));
  CUDA_TRY(cudaMemcpyAsync(dq, B[7].p, bq, cudaMemcpyDeviceToHost, dn));
  CUDA_TRY(cudaMemcpyAsync(dk_out, B[8].p, bq, cudaMemcpyDeviceToHost, dn));
  CUDA_TRY(cudaMemcpyAsync(dv_out, B[10].p, bv, cudaMemcpyDeviceToHost, dn));
  if (dbias && E) CUDA_TRY(cudaMemcpyAsync(dbias, B[5].p, E * as, cudaMemcpyDeviceToHost, dn));
  CUDA_TRY(cudaEventRecord(c->d2h_done[sidx], dn));  // this set's outputs read back
  c->pending = true;
  if (!sync) return GTE_OK;
  CUDA_TRY(cudaStreamSynchronize(dn));
  c->pending = false;
  return drain_errors(c);
}

int gte_sparse_attn_fwd_bwd_host(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                                 const void* q, const void* k, const void* v, const void* dout,
                                 const void* bias, void* out, void* dq, void* dk_out, void* dv_out,
                                 void* dbias) {
  return fwd_bwd_host_impl(c, plan, dtype, H, dk, dv, q, k, v, dout, bias, out, dq, dk_out, dv_out, dbias, true);
}

int gte_sparse_attn_fwd_bwd_host_async(gte_ctx* c, const gte_plan* plan, int dtype, int H, int dk, int dv,
                                       const void* q, const void* k, const void* v, const void* dout,
                                       const void* bias, void* out, void* dq, void* dk_out, void* dv_out,
                                       void* dbias) {
  return fwd_bwd_host_impl(c, plan, dtype, H, dk, dv, q, k, v, dout, bias, out, dq, dk_out, dv_out, dbias, false);
}

}  // extern "C"

namespace gte_b200 {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
int64_t& ctx_launch_counter(gte_ctx* c) { return c->launches; }
void* ctx_stream(gte_ctx* c) { return (void*)c->stream; }
int ctx_device(gte_ctx* c) { return c->device; }
// grow-only device workspace owned by the context (stream-ordered use only)
void* ctx_scratch(gte_ctx* c, size_t bytes) { return c->scratch.ensure(bytes) == cudaSuccess ? c->scratch.p : nullptr; }

cudaError_t launch_finite_rows(int dtype, const void* k, const void* v, const int32_t* rows, int nrows,
                               int64_t ldq, int64_t ldv, int64_t wq, int64_t wv, int* err, cudaStream_t st) {
  const unsigned grid = nrows < 4096 ? (unsigned)nrows : 4096u;
  switch (dtype) {
    case GTE_F64:
      finite_rows_kernel<double><<<grid, 64, 0, st>>>((const double*)k, (const double*)v, rows, nrows, ldq, ldv, wq, wv, err);
      break;
    case GTE_F32:
      finite_rows_kernel<float><<<grid, 64, 0, st>>>((const float*)k, (const float*)v, rows, nrows, ldq, ldv, wq, wv, err);
      break;
    default:
      finite_rows_kernel<__nv_bfloat16><<<grid, 64, 0, st>>>((const __nv_bfloat16*)k, (const __nv_bfloat16*)v, rows,
                                                              nrows, ldq, ldv, wq, wv, err);
  }
  return cudaGetLastError();
}
}  // namespace gte_b200

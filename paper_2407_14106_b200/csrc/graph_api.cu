// Graph/CSR builders, cluster grid and Elastic-Computation-Reformation layout
// on the GPU (C ABI part 2, include/gte_b200.h).
//
// Reference functions replaced (bit-exact outputs):
//   graph_from_edges   proj/src/graph.cpp:49-66       -> radix sort of (u*n+v) keys + unique + scan
//   add_self_loops     proj/src/graph.cpp:127-149     -> count + scan + merge-insert per row
//   permute_graph      proj/src/partition.cpp:435-456 -> relabel + graph_from_edges
//   build_cluster_grid proj/src/partition.cpp:514-539 -> smem-privatised k x k histogram, fp64 densities
//   build_layout       proj/src/reformation.cpp:111-195 -> fp64 classification (host), exact packer
//                      (pack.cpp, threads over cells), pattern materialised by count + scan + fill kernels
//   reorder            proj/src/partition.cpp:413-433 -> bisection.cpp (host greedy) +
//                      partition_gpu.cu (device coarsening / splitting)
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/gte_b200.h"
#include "pack.h"
#include "bisection.h"

// error channel shared with capi.cu
namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define GCUDA(expr)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                 \
  } while (0)

namespace {

unsigned grid_of(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (unsigned)g;
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t s) {
    st = s;
    return cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), s);
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

__global__ void range_check_kernel(const int32_t* __restrict__ s, const int32_t* __restrict__ d, int64_t m,
                                   int64_t n, unsigned long long* first_bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    if (s[i] < 0 || s[i] >= n || d[i] < 0 || d[i] >= n) atomicMin(first_bad, (unsigned long long)i);
}

__global__ void make_keys_kernel(const int32_t* __restrict__ s, const int32_t* __restrict__ d, int64_t m, int64_t n,
                                 uint64_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (uint64_t)s[i] * (uint64_t)n + (uint64_t)d[i];
}

__global__ void keys_to_csr_kernel(const uint64_t* __restrict__ keys, int64_t nnz, int64_t n, int32_t* __restrict__ cols,
                                   int32_t* __restrict__ counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    cols[i] = (int32_t)(k % (uint64_t)n);
    atomicAdd(counts + (k / (uint64_t)n), 1);
  }
}

__global__ void relabel_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols, int64_t n,
                               const int32_t* __restrict__ f, int32_t* __restrict__ s, int32_t* __restrict__ d) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int32_t fu = f[w];
  for (int e = row_ptr[w] + lane; e < row_ptr[w + 1]; e += 32) {
    s[e] = fu;
    d[e] = f[cols[e]];
  }
}

__global__ void loop_count_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols, int64_t n,
                                  int32_t* __restrict__ cnt) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int b = row_ptr[u], e = row_ptr[u + 1];
    // cols sorted: binary search for u
    int lo = b, hi = e;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cols[mid] < u) lo = mid + 1; else hi = mid;
    }
    const bool has = lo < e && cols[lo] == u;
    cnt[u] = (e - b) + (has ? 0 : 1);
  }
}

__global__ void loop_fill_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols, int64_t n,
                                 const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_cols) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int b = row_ptr[u], e = row_ptr[u + 1];
    int w = out_ptr[u];
    bool placed = false;
    for (int i = b; i < e; ++i) {
      const int v = cols[i];
      if (!placed && v >= u) {  // graph.cpp:139-142
        if (v != u) out_cols[w++] = (int32_t)u;
        placed = true;
      }
      out_cols[w++] = v;
    }
    if (!placed) out_cols[w++] = (int32_t)u;
  }
}

__device__ __forceinline__ int64_t cluster_of_dev(int64_t pos, int64_t n, int64_t k) {
  const int64_t base = n / k, rem = n % k, cut = rem * (base + 1);
  return pos < cut ? pos / (base + 1) : rem + (pos - cut) / base;  // partition.cpp:502-508
}

__global__ void grid_hist_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols, int64_t n,
                                 const int32_t* __restrict__ f, int64_t k, unsigned long long* __restrict__ out) {
  extern __shared__ unsigned long long hist[];
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const int64_t a = cluster_of_dev(f ? f[u] : u, n, k);
    for (int e = row_ptr[u] + lane; e < row_ptr[u + 1]; e += 32) {
      const int64_t v = cols[e];
      atomicAdd(&hist[a * k + cluster_of_dev(f ? f[v] : v, n, k)], 1ULL);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * k; i += blockDim.x)
    if (hist[i]) atomicAdd(out + i, hist[i]);
}

// Layout pattern materialisation. Row u of cluster a visits cells b = 0..k-1:
// untouched -> its neighbours inside [bnd_b, bnd_b+1) (binary search in the
// sorted row), transferred -> the column spans of the tiles crossing the
// row (host-built per-row list, sorted by (b, col)). reformation.cpp:162-193
struct LayoutDev {
  int64_t n, k, d_b;
  const int64_t* bnd;          // k+1
  const int32_t* cell_state;   // k*k
  const int32_t* row_ptr;      // permuted graph
  const int32_t* cols;
  const int32_t* rt_ptr;       // n+1: per-row tile list offsets
  const int32_t* rt_cell_b;    // cell column index b of each tile entry
  const int32_t* rt_col;       // global first column of each tile entry
};

__device__ __forceinline__ int lower_bound_dev(const int32_t* a, int lo, int hi, int64_t x) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool kFill>
__global__ void layout_rows_kernel(LayoutDev L, int32_t* __restrict__ counts, const int32_t* __restrict__ out_ptr,
                                   int32_t* __restrict__ out_cols) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < L.n; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = cluster_of_dev(u, L.n, L.k);
    const int rb = L.row_ptr[u], re = L.row_ptr[u + 1];
    int t = L.rt_ptr[u];
    const int te = L.rt_ptr[u + 1];
    int64_t w = kFill ? out_ptr[u] : 0;
    for (int64_t b = 0; b < L.k; ++b) {
      if (L.cell_state[a * L.k + b] == 0) {
        const int lo = lower_bound_dev(L.cols, rb, re, L.bnd[b]);
        const int hi = lower_bound_dev(L.cols, lo, re, L.bnd[b + 1]);
        if (kFill)
          for (int i = lo; i < hi; ++i) out_cols[w++] = L.cols[i];
        else
          w += hi - lo;
      } else {
        while (t < te && L.rt_cell_b[t] == b) {
          if (kFill)
            for (int64_t c = 0; c < L.d_b; ++c) out_cols[w++] = (int32_t)(L.rt_col[t] + c);
          else
            w += L.d_b;
          ++t;
        }
      }
    }
    if (!kFill) counts[u] = (int32_t)w;
  }
}

int csr_from_keys(gte_ctx* c, cudaStream_t st, uint64_t* keys, int64_t m, int64_t n, int32_t* d_row_ptr,
                  int32_t* d_cols, int64_t* nnz_out) {
  int bits = 1;
  const unsigned __int128 maxkey = (unsigned __int128)n * (unsigned __int128)n;
  while (bits < 64 && ((unsigned __int128)1 << bits) < maxkey) ++bits;
  DBuf<uint64_t> sorted, uniq;
  DBuf<int> nsel;
  DBuf<int32_t> counts;
  GCUDA(sorted.alloc(m, st));
  GCUDA(uniq.alloc(m, st));
  GCUDA(nsel.alloc(1, st));
  GCUDA(counts.alloc(n + 1, st));
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, sorted.p, (int)m, 0, bits, st);
  cub::DeviceSelect::Unique(nullptr, b2, sorted.p, uniq.p, nsel.p, (int)m, st);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, counts.p, d_row_ptr, (int)(n + 1), st);
  size_t tb = std::max(b1, std::max(b2, b3));
  DBuf<char> tmp;
  GCUDA(tmp.alloc(tb + 16, st));
  if (m > 0) {
    size_t t = tb;
    GCUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t, keys, sorted.p, (int)m, 0, bits, st));
    t = tb;
    GCUDA(cub::DeviceSelect::Unique(tmp.p, t, sorted.p, uniq.p, nsel.p, (int)m, st));
  } else {
    GCUDA(cudaMemsetAsync(nsel.p, 0, sizeof(int), st));
  }
  int h_n = 0;
  GCUDA(cudaMemcpyAsync(&h_n, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  GCUDA(cudaMemsetAsync(counts.p, 0, sizeof(int32_t) * (n + 1), st));
  keys_to_csr_kernel<<<grid_of(h_n), 256, 0, st>>>(uniq.p, h_n, n, d_cols, counts.p);
  size_t t = tb;
  GCUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, counts.p, d_row_ptr, (int)(n + 1), st));
  ctx_launch_counter(c) += 4;
  *nnz_out = h_n;
  GCUDA(cudaStreamSynchronize(st));
  return GTE_OK;
}

}  // namespace

struct gte_layout {
  int64_t n = 0, k = 0, d_b = 0, dropped = 0, nnz = 0;
  std::vector<int32_t> cell_state;
  std::vector<int64_t> block_off, blocks;
  int32_t* row_ptr = nullptr;  // device pattern
  int32_t* cols = nullptr;
};

extern "C" {

int gte_graph_from_edges(gte_ctx* c, int64_t n, int64_t m, const int32_t* d_src, const int32_t* d_dst,
                         int32_t* d_row_ptr, int32_t* d_cols, int64_t* nnz_out) {
  if (n < 0) return set_error(GTE_DATA, "graph_from_edges: negative node count");
  if (n >= INT_MAX || m >= INT_MAX) return set_error(GTE_CONFIG, "graph_from_edges: exceeds int32 device index range");
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  DBuf<unsigned long long> bad;
  GCUDA(bad.alloc(1, st));
  const unsigned long long init = ~0ULL;
  GCUDA(cudaMemcpyAsync(bad.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
  if (m > 0) range_check_kernel<<<grid_of(m), 256, 0, st>>>(d_src, d_dst, m, n, bad.p);
  unsigned long long first = 0;
  GCUDA(cudaMemcpyAsync(&first, bad.p, sizeof first, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  if (first != ~0ULL) {
    int32_t uv[2];
    GCUDA(cudaMemcpy(&uv[0], d_src + first, 4, cudaMemcpyDeviceToHost));
    GCUDA(cudaMemcpy(&uv[1], d_dst + first, 4, cudaMemcpyDeviceToHost));
    const int32_t badv = (uv[0] < 0 || uv[0] >= n) ? uv[0] : uv[1];
    return set_error(GTE_DATA, "graph_from_edges: node id " + std::to_string(badv) + " out of range [0, " +
                                   std::to_string(n) + ")");
  }
  DBuf<uint64_t> keys;
  GCUDA(keys.alloc(m, st));
  make_keys_kernel<<<grid_of(m), 256, 0, st>>>(d_src, d_dst, m, n, keys.p);
  ctx_launch_counter(c) += 2;
  return csr_from_keys(c, st, keys.p, m, n, d_row_ptr, d_cols, nnz_out);
}

int gte_add_self_loops(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                       int32_t* d_out_row_ptr, int32_t* d_out_cols, int64_t* nnz_out) {
  (void)nnz;
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  DBuf<int32_t> cnt;
  GCUDA(cnt.alloc(n + 1, st));
  GCUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (n + 1), st));
  loop_count_kernel<<<grid_of(n), 256, 0, st>>>(d_row_ptr, d_cols, n, cnt.p);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, d_out_row_ptr, (int)(n + 1), st);
  DBuf<char> tmp;
  GCUDA(tmp.alloc(tb + 16, st));
  GCUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, d_out_row_ptr, (int)(n + 1), st));
  loop_fill_kernel<<<grid_of(n), 256, 0, st>>>(d_row_ptr, d_cols, n, d_out_row_ptr, d_out_cols);
  ctx_launch_counter(c) += 3;
  int32_t tot = 0;
  GCUDA(cudaMemcpyAsync(&tot, d_out_row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  *nnz_out = tot;
  return GTE_OK;
}

int gte_reorder(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, int64_t k, uint64_t seed,
                int64_t* forward, int64_t* inverse) {
  (void)nnz;
  // partition.cpp:414-415
  if (k < 1 || (k & (k - 1)) != 0) return set_error(GTE_CONFIG, "reorder: k must be a power of two >= 1");
  if (k > n) return set_error(GTE_CONFIG, "reorder: k exceeds node count");
  try {
    reorder_cluster(n, row_off, cols, k, seed, forward, inverse);
  } catch (const std::exception& e) {
    return set_error(GTE_CUDA, e.what());
  }
  return GTE_OK;
}

int gte_permute_graph(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                      const int64_t* forward, int32_t* d_out_row_ptr, int32_t* d_out_cols) {
  // permutation validity (partition.cpp:436)
  std::vector<char> seen(n, 0);
  std::vector<int32_t> f32(n > 0 ? n : 1);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t f = forward[i];
    if (f < 0 || f >= n || seen[f]) return set_error(GTE_CONFIG, "permute_graph: bad permutation");
    seen[f] = 1;
    f32[i] = (int32_t)f;
  }
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  DBuf<int32_t> df, s, d;
  GCUDA(df.alloc(n, st));
  GCUDA(s.alloc(nnz, st));
  GCUDA(d.alloc(nnz, st));
  GCUDA(cudaMemcpyAsync(df.p, f32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  if (n > 0) relabel_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(d_row_ptr, d_cols, n, df.p, s.p, d.p);
  ctx_launch_counter(c) += 1;
  int64_t out_nnz = 0;
  DBuf<uint64_t> keys;
  GCUDA(keys.alloc(nnz, st));
  make_keys_kernel<<<grid_of(nnz), 256, 0, st>>>(s.p, d.p, nnz, n, keys.p);
  int rc = csr_from_keys(c, st, keys.p, nnz, n, d_out_row_ptr, d_out_cols, &out_nnz);
  GCUDA(cudaStreamSynchronize(st));  // f32 (host) must outlive the H2D copy
  return rc;
}

int gte_cluster_boundaries(int64_t n, int64_t k, int64_t* b) {
  if (k < 1) return set_error(GTE_CONFIG, "cluster_boundaries: k must be >= 1");
  const int64_t base = n / k, rem = n % k;  // partition.cpp:495-500
  b[0] = 0;
  for (int64_t i = 0; i < k; ++i) b[i + 1] = b[i] + base + (i < rem ? 1 : 0);
  return GTE_OK;
}

int gte_build_cluster_grid(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                           const int64_t* forward, int64_t k, int64_t* bnd, int64_t* cell_nnz, double* cell_density) {
  (void)nnz;
  if (k < 1 || k > n) return set_error(GTE_CONFIG, "build_cluster_grid: invalid k");
  if (k * k * 8 > 200 * 1024) return set_error(GTE_CONFIG, "build_cluster_grid: k too large for the on-chip histogram");
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  DBuf<int32_t> df;
  std::vector<int32_t> f32;
  if (forward) {
    std::vector<char> seen(n, 0);
    f32.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t f = forward[i];
      if (f < 0 || f >= n || seen[f]) return set_error(GTE_CONFIG, "build_cluster_grid: permutation does not match graph");
      seen[f] = 1;
      f32[i] = (int32_t)f;
    }
    GCUDA(df.alloc(n, st));
    GCUDA(cudaMemcpyAsync(df.p, f32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  }
  DBuf<unsigned long long> hist;
  GCUDA(hist.alloc(k * k, st));
  GCUDA(cudaMemsetAsync(hist.p, 0, sizeof(unsigned long long) * k * k, st));
  const size_t smem = sizeof(unsigned long long) * k * k;
  if (smem > 48 * 1024) GCUDA(cudaFuncSetAttribute(grid_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  grid_hist_kernel<<<148 * 2, 512, smem, st>>>(d_row_ptr, d_cols, n, forward ? df.p : nullptr, k, hist.p);
  ctx_launch_counter(c) += 1;
  std::vector<unsigned long long> h(k * k);
  GCUDA(cudaMemcpyAsync(h.data(), hist.p, sizeof(unsigned long long) * k * k, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  gte_cluster_boundaries(n, k, bnd);
  for (int64_t a = 0; a < k; ++a)
    for (int64_t b = 0; b < k; ++b) {
      cell_nnz[a * k + b] = (int64_t)h[a * k + b];
      const double area = static_cast<double>(bnd[a + 1] - bnd[a]) * static_cast<double>(bnd[b + 1] - bnd[b]);
      cell_density[a * k + b] = static_cast<double>(cell_nnz[a * k + b]) / area;  // partition.cpp:533-535
    }
  return GTE_OK;
}

int gte_diagonal_edge_fraction(int64_t k, const int64_t* cell_nnz, double* out) {
  int64_t total = 0, diag = 0;
  for (int64_t i = 0; i < k * k; ++i) total += cell_nnz[i];
  if (total == 0) return set_error(GTE_DATA, "diagonal_edge_fraction: empty graph");
  for (int64_t a = 0; a < k; ++a) diag += cell_nnz[a * k + a];
  *out = static_cast<double>(diag) / static_cast<double>(total);
  return GTE_OK;
}

int gte_pack_subblocks(int64_t m, const int64_t* er, const int64_t* ec, int64_t n_rows, int64_t n_cols, int64_t d_b,
                       int64_t* tiles_rc, int64_t* ntiles) {
  *ntiles = 0;
  if (d_b < 1) return set_error(GTE_CONFIG, "pack_subblocks: d_b must be >= 1");
  if (d_b > n_rows || d_b > n_cols)
    return set_error(GTE_CONFIG, "pack_subblocks: d_b " + std::to_string(d_b) + " too large for " +
                                     std::to_string(n_rows) + "x" + std::to_string(n_cols) + " cell");
  if (m == 0) return GTE_OK;
  for (int64_t e = 0; e < m; ++e)
    if (er[e] < 0 || er[e] >= n_rows || ec[e] < 0 || ec[e] >= n_cols)
      return set_error(GTE_CONFIG, "pack_subblocks: edge outside cell");
  // the reference marks a grid, so duplicate edges count once
  std::vector<std::pair<int64_t, int64_t>> es(m);
  for (int64_t e = 0; e < m; ++e) es[e] = {er[e], ec[e]};
  std::sort(es.begin(), es.end());
  es.erase(std::unique(es.begin(), es.end()), es.end());
  std::vector<int64_t> r(es.size()), cc(es.size());
  for (size_t i = 0; i < es.size(); ++i) {
    r[i] = es[i].first;
    cc[i] = es[i].second;
  }
  // want counts the input edges (duplicates included), reformation.cpp:73-74
  std::vector<int64_t> out;
  pack_subblocks_exact(r.data(), cc.data(), (int64_t)r.size(), n_rows, n_cols, d_b, out,
                       (m + d_b * d_b - 1) / (d_b * d_b));
  *ntiles = (int64_t)out.size() / 2;
  std::copy(out.begin(), out.end(), tiles_rc);
  return GTE_OK;
}

int gte_build_layout(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols, int64_t k,
                     const int64_t* bnd, const int64_t* cell_nnz, const double* cell_density, int strategy,
                     double beta_thre, double beta_g, int64_t d_b, gte_layout** out) {
  if (bnd[k] != n) return set_error(GTE_CONFIG, "build_layout: grid/graph size mismatch");
  int64_t tot = 0;
  for (int64_t i = 0; i < k * k; ++i) tot += cell_nnz[i];
  if (tot != nnz) return set_error(GTE_CONFIG, "build_layout: grid/graph nnz mismatch");
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  const double threshold = strategy == 0 ? beta_g : beta_thre;  // reformation.cpp:119
  auto* L = new gte_layout();
  L->n = n;
  L->k = k;
  L->d_b = d_b;
  L->cell_state.assign(k * k, 0);
  for (int64_t i = 0; i < k * k; ++i)
    if (cell_density[i] < threshold) L->cell_state[i] = 1;  // reformation.cpp:143
  // host copy of the (permuted) graph for cell bucketing
  std::vector<int32_t> hro(n + 1), hco(nnz > 0 ? nnz : 1);
  GCUDA(cudaMemcpyAsync(hro.data(), d_row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (nnz) GCUDA(cudaMemcpyAsync(hco.data(), d_cols, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  // bucket edges of transferred cells in cell-local coordinates (CSR order)
  std::vector<std::vector<int64_t>> er(k * k), ec(k * k);
  for (int64_t u = 0; u < n; ++u) {
    int64_t a = 0;
    while (bnd[a + 1] <= u) ++a;
    for (int32_t e = hro[u]; e < hro[u + 1]; ++e) {
      const int64_t v = hco[e];
      const int64_t b = std::upper_bound(bnd, bnd + k + 1, v) - bnd - 1;
      if (!L->cell_state[a * k + b]) continue;
      er[a * k + b].push_back(u - bnd[a]);
      ec[a * k + b].push_back(v - bnd[b]);
    }
  }
  // d_b validation in cell order (the reference throws at the first failing cell)
  for (int64_t a = 0; a < k; ++a)
    for (int64_t b = 0; b < k; ++b) {
      const int64_t cell = a * k + b;
      if (!L->cell_state[cell] || er[cell].empty()) continue;
      const int64_t nr = bnd[a + 1] - bnd[a], nc = bnd[b + 1] - bnd[b];
      if (d_b < 1 || d_b > nr || d_b > nc) {
        delete L;
        if (d_b < 1) return set_error(GTE_CONFIG, "pack_subblocks: d_b must be >= 1");
        return set_error(GTE_CONFIG, "pack_subblocks: d_b " + std::to_string(d_b) + " too large for " +
                                         std::to_string(nr) + "x" + std::to_string(nc) + " cell");
      }
    }
  std::vector<std::vector<int64_t>> tiles(k * k);
  {
    std::vector<int64_t> work;
    for (int64_t cell = 0; cell < k * k; ++cell)
      if (L->cell_state[cell] && !er[cell].empty()) work.push_back(cell);
    std::sort(work.begin(), work.end(), [&](int64_t x, int64_t y) { return er[x].size() > er[y].size(); });
    std::atomic<size_t> next{0};
    const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)work.size()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nth; ++t)
      pool.emplace_back([&] {
        for (size_t i = next++; i < work.size(); i = next++) {
          const int64_t cell = work[i], a = cell / k, b = cell % k;
          pack_subblocks_exact(er[cell].data(), ec[cell].data(), (int64_t)er[cell].size(), bnd[a + 1] - bnd[a],
                               bnd[b + 1] - bnd[b], d_b, tiles[cell]);
        }
      });
    for (auto& th : pool) th.join();
  }
  // dropped edges: not inside any tile of their cell (reformation.cpp:147-157)
  L->block_off.assign(k * k + 1, 0);
  for (int64_t cell = 0; cell < k * k; ++cell) {
    const auto& t = tiles[cell];
    const int64_t nt = (int64_t)t.size() / 2;
    L->block_off[cell + 1] = L->block_off[cell] + nt;
    if (er[cell].empty()) continue;
    // row -> tiles crossing it
    std::vector<std::pair<int64_t, int64_t>> spans;  // (row_start, col_start)
    for (int64_t i = 0; i < nt; ++i) spans.emplace_back(t[2 * i], t[2 * i + 1]);
    std::sort(spans.begin(), spans.end());
    int64_t covered = 0;
    for (size_t e = 0; e < er[cell].size(); ++e) {
      const int64_t r = er[cell][e], cc = ec[cell][e];
      for (auto& [tr, tc] : spans) {
        if (tr > r) break;
        if (r < tr + d_b && cc >= tc && cc < tc + d_b) {
          ++covered;
          break;
        }
      }
    }
    L->dropped += (int64_t)er[cell].size() - covered;
  }
  L->blocks.reserve(2 * L->block_off[k * k]);
  for (int64_t cell = 0; cell < k * k; ++cell) L->blocks.insert(L->blocks.end(), tiles[cell].begin(), tiles[cell].end());
  // per-row tile lists sorted by (cell column b, col)
  std::vector<int32_t> rt_cnt(n + 1, 0);
  for (int64_t cell = 0; cell < k * k; ++cell) {
    const int64_t a = cell / k;
    for (size_t i = 0; i < tiles[cell].size(); i += 2)
      for (int64_t r = tiles[cell][i]; r < tiles[cell][i] + d_b; ++r) rt_cnt[bnd[a] + r + 1]++;
  }
  for (int64_t u = 0; u < n; ++u) rt_cnt[u + 1] += rt_cnt[u];
  const int32_t nrt = rt_cnt[n];
  std::vector<int32_t> rt_b(nrt > 0 ? nrt : 1), rt_col(nrt > 0 ? nrt : 1), fillp(rt_cnt.begin(), rt_cnt.end() - 1);
  for (int64_t cell = 0; cell < k * k; ++cell) {
    const int64_t a = cell / k, b = cell % k;
    for (size_t i = 0; i < tiles[cell].size(); i += 2)
      for (int64_t r = tiles[cell][i]; r < tiles[cell][i] + d_b; ++r) {
        const int32_t pos = fillp[bnd[a] + r]++;
        rt_b[pos] = (int32_t)b;
        rt_col[pos] = (int32_t)(bnd[b] + tiles[cell][i + 1]);
      }
  }
  for (int64_t u = 0; u < n; ++u) {
    // sort this row's entries by (b, col)
    std::vector<std::pair<int32_t, int32_t>> tmp;
    for (int32_t i = rt_cnt[u]; i < rt_cnt[u + 1]; ++i) tmp.emplace_back(rt_b[i], rt_col[i]);
    if (tmp.size() < 2) continue;
    std::sort(tmp.begin(), tmp.end());
    for (size_t i = 0; i < tmp.size(); ++i) {
      rt_b[rt_cnt[u] + i] = tmp[i].first;
      rt_col[rt_cnt[u] + i] = tmp[i].second;
    }
  }
  DBuf<int64_t> dbnd;
  DBuf<int32_t> dstate, drt, drtb, drtc, dcnt;
  GCUDA(dbnd.alloc(k + 1, st));
  GCUDA(dstate.alloc(k * k, st));
  GCUDA(drt.alloc(n + 1, st));
  GCUDA(drtb.alloc(nrt, st));
  GCUDA(drtc.alloc(nrt, st));
  GCUDA(dcnt.alloc(n + 1, st));
  GCUDA(cudaMemcpyAsync(dbnd.p, bnd, sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice, st));
  GCUDA(cudaMemcpyAsync(dstate.p, L->cell_state.data(), sizeof(int32_t) * k * k, cudaMemcpyHostToDevice, st));
  GCUDA(cudaMemcpyAsync(drt.p, rt_cnt.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
  if (nrt) {
    GCUDA(cudaMemcpyAsync(drtb.p, rt_b.data(), sizeof(int32_t) * nrt, cudaMemcpyHostToDevice, st));
    GCUDA(cudaMemcpyAsync(drtc.p, rt_col.data(), sizeof(int32_t) * nrt, cudaMemcpyHostToDevice, st));
  }
  LayoutDev LD{n, k, d_b, dbnd.p, dstate.p, d_row_ptr, d_cols, drt.p, drtb.p, drtc.p};
  GCUDA(cudaMemsetAsync(dcnt.p, 0, sizeof(int32_t) * (n + 1), st));
  GCUDA(cudaMallocAsync(&L->row_ptr, sizeof(int32_t) * (n + 1), st));
  layout_rows_kernel<false><<<grid_of(n), 256, 0, st>>>(LD, dcnt.p, nullptr, nullptr);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, dcnt.p, L->row_ptr, (int)(n + 1), st);
  DBuf<char> tmp;
  GCUDA(tmp.alloc(tb + 16, st));
  GCUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, dcnt.p, L->row_ptr, (int)(n + 1), st));
  int32_t total = 0;
  GCUDA(cudaMemcpyAsync(&total, L->row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  L->nnz = total;
  GCUDA(cudaMallocAsync(&L->cols, sizeof(int32_t) * (total + 1), st));
  layout_rows_kernel<true><<<grid_of(n), 256, 0, st>>>(LD, nullptr, L->row_ptr, L->cols);
  ctx_launch_counter(c) += 3;
  GCUDA(cudaStreamSynchronize(st));
  *out = L;
  return GTE_OK;
}

int gte_layout_info(const gte_layout* L, int64_t* transferred, int64_t* n_blocks, int64_t* dropped, int64_t* pattern_nnz) {
  if (transferred) {
    int64_t t = 0;
    for (int32_t s : L->cell_state) t += s;
    *transferred = t;
  }
  if (n_blocks) *n_blocks = L->block_off.back();
  if (dropped) *dropped = L->dropped;
  if (pattern_nnz) *pattern_nnz = L->nnz;
  return GTE_OK;
}

int gte_layout_cells(const gte_layout* L, int32_t* cell_state, int64_t* block_off, int64_t* blocks) {
  std::copy(L->cell_state.begin(), L->cell_state.end(), cell_state);
  std::copy(L->block_off.begin(), L->block_off.end(), block_off);
  std::copy(L->blocks.begin(), L->blocks.end(), blocks);
  return GTE_OK;
}

int gte_layout_pattern_device(const gte_layout* L, const int32_t** d_row_ptr, const int32_t** d_cols) {
  *d_row_ptr = L->row_ptr;
  *d_cols = L->cols;
  return GTE_OK;
}

int gte_layout_pattern_host(const gte_layout* L, int64_t* row_off, int64_t* cols) {
  std::vector<int32_t> ro(L->n + 1), co(L->nnz > 0 ? L->nnz : 1);
  GCUDA(cudaMemcpy(ro.data(), L->row_ptr, sizeof(int32_t) * (L->n + 1), cudaMemcpyDeviceToHost));
  if (L->nnz) GCUDA(cudaMemcpy(co.data(), L->cols, sizeof(int32_t) * L->nnz, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i <= L->n; ++i) row_off[i] = ro[i];
  for (int64_t i = 0; i < L->nnz; ++i) cols[i] = co[i];
  return GTE_OK;
}

int gte_layout_destroy(gte_layout* L) {
  if (!L) return GTE_OK;
  cudaDeviceSynchronize();
  cudaFree(L->row_ptr);
  cudaFree(L->cols);
  delete L;
  return GTE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host-pointer twins (int64 reference CSR in host memory).
namespace {

struct HostCsr32 {
  DBuf<int32_t> rp, cl;
  int alloc_copy(int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols, cudaStream_t st) {
    std::vector<int32_t> r(n + 1), c(nnz > 0 ? nnz : 1);
    for (int64_t i = 0; i <= n; ++i) r[i] = (int32_t)row_off[i];
    for (int64_t i = 0; i < nnz; ++i) c[i] = (int32_t)cols[i];
    GCUDA(rp.alloc(n + 1, st));
    GCUDA(cl.alloc(nnz, st));
    GCUDA(cudaMemcpyAsync(rp.p, r.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, st));
    if (nnz) GCUDA(cudaMemcpyAsync(cl.p, c.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
    GCUDA(cudaStreamSynchronize(st));
    return GTE_OK;
  }
};

int d2h_csr(int64_t n, int64_t nnz, const int32_t* d_rp, const int32_t* d_cl, int64_t* row_off, int64_t* cols,
            cudaStream_t st) {
  std::vector<int32_t> r(n + 1), c(nnz > 0 ? nnz : 1);
  GCUDA(cudaMemcpyAsync(r.data(), d_rp, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st));
  if (nnz) GCUDA(cudaMemcpyAsync(c.data(), d_cl, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
  GCUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i <= n; ++i) row_off[i] = r[i];
  for (int64_t i = 0; i < nnz; ++i) cols[i] = c[i];
  return GTE_OK;
}

}  // namespace

extern "C" {

int gte_graph_from_edges_host(gte_ctx* c, int64_t n, int64_t m, const int64_t* src, const int64_t* dst,
                              int64_t* row_off, int64_t* cols, int64_t* nnz_out) {
  if (n < 0) return set_error(GTE_DATA, "graph_from_edges: negative node count");
  for (int64_t e = 0; e < m; ++e) {  // graph.cpp:51-54, first offending endpoint in edge order
    if (src[e] < 0 || src[e] >= n)
      return set_error(GTE_DATA, "graph_from_edges: node id " + std::to_string(src[e]) + " out of range [0, " +
                                     std::to_string(n) + ")");
    if (dst[e] < 0 || dst[e] >= n)
      return set_error(GTE_DATA, "graph_from_edges: node id " + std::to_string(dst[e]) + " out of range [0, " +
                                     std::to_string(n) + ")");
  }
  if (n >= INT_MAX || m >= INT_MAX) return set_error(GTE_CONFIG, "graph_from_edges: exceeds int32 device index range");
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  std::vector<int32_t> s(m > 0 ? m : 1), d(m > 0 ? m : 1);
  for (int64_t e = 0; e < m; ++e) {
    s[e] = (int32_t)src[e];
    d[e] = (int32_t)dst[e];
  }
  DBuf<int32_t> ds, dd, rp, cl;
  GCUDA(ds.alloc(m, st));
  GCUDA(dd.alloc(m, st));
  GCUDA(rp.alloc(n + 1, st));
  GCUDA(cl.alloc(m, st));
  GCUDA(cudaMemcpyAsync(ds.p, s.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
  GCUDA(cudaMemcpyAsync(dd.p, d.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
  int rc = gte_graph_from_edges(c, n, m, ds.p, dd.p, rp.p, cl.p, nnz_out);
  if (rc) return rc;
  return d2h_csr(n, *nnz_out, rp.p, cl.p, row_off, cols, st);
}

int gte_add_self_loops_host(gte_ctx* c, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                            int64_t* out_row_off, int64_t* out_cols, int64_t* nnz_out) {
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  HostCsr32 in;
  int rc = in.alloc_copy(n, nnz, row_off, cols, st);
  if (rc) return rc;
  DBuf<int32_t> rp, cl;
  GCUDA(rp.alloc(n + 1, st));
  GCUDA(cl.alloc(nnz + n, st));
  rc = gte_add_self_loops(c, n, nnz, in.rp.p, in.cl.p, rp.p, cl.p, nnz_out);
  if (rc) return rc;
  return d2h_csr(n, *nnz_out, rp.p, cl.p, out_row_off, out_cols, st);
}

int gte_permute_graph_host(gte_ctx* c, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                           const int64_t* forward, int64_t* out_row_off, int64_t* out_cols) {
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  HostCsr32 in;
  int rc = in.alloc_copy(n, nnz, row_off, cols, st);
  if (rc) return rc;
  DBuf<int32_t> rp, cl;
  GCUDA(rp.alloc(n + 1, st));
  GCUDA(cl.alloc(nnz, st));
  rc = gte_permute_graph(c, n, nnz, in.rp.p, in.cl.p, forward, rp.p, cl.p);
  if (rc) return rc;
  return d2h_csr(n, nnz, rp.p, cl.p, out_row_off, out_cols, st);
}

int gte_build_cluster_grid_host(gte_ctx* c, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                                const int64_t* forward, int64_t k, int64_t* bnd, int64_t* cell_nnz,
                                double* cell_density) {
  if (k < 1 || k > n) return set_error(GTE_CONFIG, "build_cluster_grid: invalid k");
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  HostCsr32 in;
  int rc = in.alloc_copy(n, nnz, row_off, cols, st);
  if (rc) return rc;
  return gte_build_cluster_grid(c, n, nnz, in.rp.p, in.cl.p, forward, k, bnd, cell_nnz, cell_density);
}

int gte_build_layout_host(gte_ctx* c, int64_t n, int64_t nnz, const int64_t* row_off, const int64_t* cols,
                          int64_t k, const int64_t* bnd, const int64_t* cell_nnz, const double* cell_density,
                          int strategy, double beta_thre, double beta_g, int64_t d_b, gte_layout** out) {
  cudaStream_t st = (cudaStream_t)ctx_stream(c);
  HostCsr32 in;
  int rc = in.alloc_copy(n, nnz, row_off, cols, st);
  if (rc) return rc;
  return gte_build_layout(c, n, nnz, in.rp.p, in.cl.p, k, bnd, cell_nnz, cell_density, strategy, beta_thre, beta_g,
                          d_b, out);
}

}  // extern "C"

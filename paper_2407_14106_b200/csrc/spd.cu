// Shortest-path-distance buckets on the GPU (reference
// SpdTable / spd_table, proj/src/graph.cpp:208-261, proj/include/gte/graph.hpp:56-74,
// consumed by the Trainer's bucket rule proj/src/model.cpp:407-423, 447-463).
//
// The reference runs one BFS per source on the host and refuses graphs above
// 20,000 nodes. Here:
//   * gte_spd_table: the same capped BFS from every source, one CTA per
//     source (visited bitmap in shared memory, queue in a per-CTA global
//     slot), two sweeps (ball sizes -> scan -> sorted fill), so the table is
//     the reference's CSR (columns ascending, uint16 distances) at any size
//     whose table fits in memory.
//   * gte_spd_pairs: distances of an arbitrary pair list without the full
//     table (what the pattern buckets need at C2-C5, where a table capped at
//     8 hops would hold every pair): the radius-2 balls B2(v) (the table at
//     cap 2) answer d <= 2 by binary search and d in {3, 4} by a min-plus
//     meet in the middle over B2(i) and B2(j) (any path of length <= 4 has a
//     midpoint within 2 of both ends; no common node means d >= 5); the rare
//     pairs left are resolved by an early-exit BFS from their source.
// Distances beyond the cap (or unreachable) map to cap + 1, as
// SpdTable::unreachable_bucket.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gte_b200.h"

namespace gte_b200 {
int set_error(int code, const std::string& msg);
int64_t& ctx_launch_counter(gte_ctx* c);
void* ctx_stream(gte_ctx* c);
}  // namespace gte_b200

using namespace gte_b200;

#define SPCUDA(expr)                                                                                  \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return set_error(GTE_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                     ":" + std::to_string(__LINE__));                                 \
  } while (0)

struct gte_spd {
  int64_t n = 0, max_dist = 0, total = 0;
  int64_t* row_off = nullptr;  // device [n + 1]
  int32_t* cols = nullptr;     // device [total]
  uint16_t* dist = nullptr;    // device [total]
};

namespace {

constexpr int kBfsThreads = 256;
constexpr uint64_t kNoKey = ~0ull;

template <typename T>
struct Scratch {  // stream-ordered device buffer
  T* p = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t s) {
    st = s;
    return cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), s);
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

// ---------------------------------------------------------------- undirected adjacency
__global__ void owner_kernel(const int32_t* __restrict__ rp, int32_t n, int32_t* __restrict__ owner) {
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n)
    for (int32_t a = rp[u]; a < rp[u + 1]; ++a) owner[a] = u;
}
__global__ void arc_keys_kernel(const int32_t* __restrict__ owner, const int32_t* __restrict__ cols, int32_t m,
                                uint64_t* __restrict__ keys) {
  const int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const uint64_t u = (uint32_t)owner[a], v = (uint32_t)cols[a];
  keys[2 * (int64_t)a] = u == v ? kNoKey : (u << 32 | v);
  keys[2 * (int64_t)a + 1] = u == v ? kNoKey : (v << 32 | u);
}
__global__ void key_split_kernel(const uint64_t* __restrict__ keys, int64_t r, int32_t* __restrict__ adj,
                                 int32_t* __restrict__ deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  adj[i] = (int32_t)(keys[i] & 0xffffffffu);
  atomicAdd(deg + (keys[i] >> 32), 1);
}

struct UAdj {
  int32_t n = 0;
  int64_t m = 0;
  Scratch<int32_t> off, adj;
};

// graph.cpp undirected_adjacency: both arc directions, no self loops, unique
cudaError_t build_uadj(cudaStream_t st, int32_t n, int32_t m, const int32_t* rp, const int32_t* cols, UAdj& u) {
  u.n = n;
  cudaError_t e;
  Scratch<int32_t> owner, deg;
  Scratch<uint64_t> keys, sorted, uniq;
  Scratch<int32_t> nuniq;
  if ((e = owner.alloc(m, st)) || (e = keys.alloc(2 * (size_t)m, st)) || (e = sorted.alloc(2 * (size_t)m, st)) ||
      (e = uniq.alloc(2 * (size_t)m, st)) || (e = nuniq.alloc(1, st)) || (e = deg.alloc(n + 1, st)) ||
      (e = u.off.alloc(n + 1, st)))
    return e;
  if (n > 0) owner_kernel<<<(n + 255) / 256, 256, 0, st>>>(rp, n, owner.p);
  if (m > 0) arc_keys_kernel<<<(m + 255) / 256, 256, 0, st>>>(owner.p, cols, m, keys.p);
  const int items = 2 * m;
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, keys.p, sorted.p, items, 0, 64, st);
  cub::DeviceSelect::Unique(nullptr, b2, sorted.p, uniq.p, nuniq.p, items, st);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, deg.p, u.off.p, n + 1, st);
  Scratch<unsigned char> tmp;
  if ((e = tmp.alloc(std::max(b1, std::max(b2, b3)) + 16, st))) return e;
  int32_t r = 0;
  if (items > 0) {
    if ((e = cub::DeviceRadixSort::SortKeys(tmp.p, b1, keys.p, sorted.p, items, 0, 64, st))) return e;
    if ((e = cub::DeviceSelect::Unique(tmp.p, b2, sorted.p, uniq.p, nuniq.p, items, st))) return e;
    if ((e = cudaMemcpyAsync(&r, nuniq.p, 4, cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    if (r > 0) {
      uint64_t last = 0;
      if ((e = cudaMemcpyAsync(&last, uniq.p + r - 1, 8, cudaMemcpyDeviceToHost, st))) return e;
      if ((e = cudaStreamSynchronize(st))) return e;
      if (last == kNoKey) --r;
    }
  }
  u.m = r;
  if ((e = u.adj.alloc(r, st))) return e;
  if ((e = cudaMemsetAsync(deg.p, 0, sizeof(int32_t) * (n + 1), st))) return e;
  if (r > 0) key_split_kernel<<<(r + 255) / 256, 256, 0, st>>>(uniq.p, r, u.adj.p, deg.p);
  if ((e = cub::DeviceScan::ExclusiveSum(tmp.p, b3, deg.p, u.off.p, n + 1, st))) return e;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- capped BFS, one CTA per source
struct BfsArgs {
  int32_t n = 0, cap = 0;
  const int32_t* off = nullptr;
  const int32_t* adj = nullptr;
  const int32_t* srcs = nullptr;  // sources (mode table: null = 0..n-1)
  int32_t nsrc = 0;
  int32_t* queue = nullptr;       // [gridDim.x][n]
  uint8_t* dist = nullptr;        // [gridDim.x][n]
  int64_t* count = nullptr;       // mode 0: ball size per source
  const int64_t* out_off = nullptr;  // mode 1: row offsets
  int32_t* out_cols = nullptr;
  uint16_t* out_dist = nullptr;
  const int32_t* tgt_off = nullptr;  // mode 2: targets of source s: [tgt_off[s], tgt_off[s+1])
  const int32_t* tgt = nullptr;
  int32_t* tgt_dist = nullptr;
  // mode 3: dense bucket rows (execution coordinates) of the Trainer's dense
  // epoch: row r < s_real of out [S x S] from a BFS of original node inv[r]
  const int64_t* inv = nullptr;      // [S] execution position -> original id
  const int64_t* fwd = nullptr;      // [s_real] original id -> execution position
  int64_t S = 0, s_real = 0, global = -1;
  int32_t graph_n = 0;
  uint8_t* rows_out = nullptr;
};

// MODE 0: ball sizes; 1: sorted (node, distance) rows; 2: distances of the targets (early exit)
template <int MODE>
__global__ void __launch_bounds__(kBfsThreads) bfs_kernel(BfsArgs a) {
  extern __shared__ uint32_t seen[];
  __shared__ int32_t s_head, s_tail, s_next, s_left;
  __shared__ int32_t s_wsum[kBfsThreads / 32];
  const int words = (a.n + 31) / 32;
  int32_t* q = a.queue + (int64_t)blockIdx.x * a.n;
  uint8_t* dd = a.dist + (int64_t)blockIdx.x * a.n;
  for (int s = blockIdx.x; s < a.nsrc; s += gridDim.x) {
    int32_t src = a.srcs ? a.srcs[s] : s;
    if (MODE == 3) {  // bucket row s: unreachable everywhere, then the BFS ball
      const int64_t i = a.inv[s];
      uint8_t* row = a.rows_out + (int64_t)s * a.S;
      const uint8_t fill = i == a.global ? 1 : (uint8_t)(a.cap + 1);  // global token: bucket 1 to all
      for (int64_t c = threadIdx.x; c < a.S; c += blockDim.x) row[c] = fill;
      __syncthreads();
      if (i == a.global || i >= a.graph_n) {
        if (threadIdx.x == 0) row[s] = 0;
        __syncthreads();
        continue;
      }
      src = (int32_t)i;
    }
    for (int w = threadIdx.x; w < words; w += blockDim.x) seen[w] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      seen[src >> 5] = 1u << (src & 31);
      q[0] = src;
      dd[src] = 0;
      s_head = 0;
      s_tail = 1;
      s_next = 1;
      s_left = MODE == 2 ? a.tgt_off[s + 1] - a.tgt_off[s] : 0;
    }
    __syncthreads();
    for (int depth = 0;; ++depth) {
      if (MODE == 2) {  // resolve the targets reached so far (first level seen = distance)
        for (int t = a.tgt_off[s] + threadIdx.x; t < a.tgt_off[s + 1]; t += blockDim.x) {
          const int32_t v = a.tgt[t];
          if (a.tgt_dist[t] < 0 && (seen[v >> 5] >> (v & 31) & 1u)) {
            a.tgt_dist[t] = dd[v];
            atomicSub(&s_left, 1);
          }
        }
        __syncthreads();
      }
      const int32_t h = s_head, t = s_tail;
      if (depth >= a.cap || h == t || (MODE == 2 && s_left == 0)) break;
      for (int32_t x = h + threadIdx.x; x < t; x += blockDim.x) {
        const int32_t u = q[x];
        for (int32_t e = a.off[u]; e < a.off[u + 1]; ++e) {
          const int32_t v = a.adj[e];
          const uint32_t bit = 1u << (v & 31);
          if (seen[v >> 5] & bit) continue;
          if (atomicOr(&seen[v >> 5], bit) & bit) continue;
          const int32_t slot = atomicAdd(&s_next, 1);
          q[slot] = v;
          dd[v] = (uint8_t)(depth + 1);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        s_head = t;
        s_tail = s_next;
      }
      __syncthreads();
    }
    if (MODE == 3) {  // scatter the ball into the row; the global token's column is bucket 1
      uint8_t* row = a.rows_out + (int64_t)s * a.S;
      for (int32_t x = threadIdx.x; x < s_next; x += blockDim.x) {
        const int32_t v = q[x];
        const int64_t c = a.fwd[v];
        if (c < a.s_real) row[c] = dd[v];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (a.global >= 0) row[a.fwd[a.global]] = 1;
        row[s] = 0;
      }
    } else if (MODE == 0) {
      if (threadIdx.x == 0) a.count[s] = s_next;
    } else if (MODE == 1) {
      // emit the visited set in node order: per-thread word ranges, block scan of popcounts
      const int per = (words + blockDim.x - 1) / blockDim.x;
      const int w0 = threadIdx.x * per, w1 = min(words, w0 + per);
      int c = 0;
      for (int w = w0; w < w1; ++w) c += __popc(seen[w]);
      int x = c;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      __syncthreads();
      int before = x - c;
      for (int w = 0; w < warp; ++w) before += s_wsum[w];
      int64_t o = a.out_off[s] + before;
      for (int w = w0; w < w1; ++w) {
        uint32_t bits = seen[w];
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int32_t v = w * 32 + b;
          a.out_cols[o] = v;
          a.out_dist[o] = dd[v];
          ++o;
        }
      }
    }
    __syncthreads();
  }
}

int bfs_grid(int32_t nsrc) { return std::max(1, std::min(nsrc, 148 * 8)); }

cudaError_t run_bfs(int mode, const BfsArgs& base, cudaStream_t st) {
  BfsArgs a = base;
  const int grid = bfs_grid(a.nsrc);
  Scratch<int32_t> q;
  Scratch<uint8_t> d;
  cudaError_t e;
  if ((e = q.alloc((size_t)grid * a.n, st)) || (e = d.alloc((size_t)grid * a.n, st))) return e;
  a.queue = q.p;
  a.dist = d.p;
  const size_t smem = sizeof(uint32_t) * ((a.n + 31) / 32);
  auto go = [&](auto kernel) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t x = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (x != cudaSuccess) return x;
    }
    kernel<<<grid, kBfsThreads, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (mode == 0) return go(bfs_kernel<0>);
  if (mode == 1) return go(bfs_kernel<1>);
  if (mode == 2) return go(bfs_kernel<2>);
  return go(bfs_kernel<3>);
}

// table = capped balls of every source (mode 0 sizes -> scan -> mode 1 rows)
int build_table(cudaStream_t st, const UAdj& u, int32_t cap, gte_spd* t) {
  t->n = u.n;
  t->max_dist = cap;
  SPCUDA(cudaMallocAsync(&t->row_off, sizeof(int64_t) * (u.n + 1), st));
  Scratch<int64_t> cnt;
  SPCUDA(cnt.alloc(u.n + 1, st));
  BfsArgs a;
  a.n = u.n;
  a.cap = cap;
  a.off = u.off.p;
  a.adj = u.adj.p;
  a.nsrc = u.n;
  a.count = cnt.p;
  SPCUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (u.n + 1), st));
  if (u.n > 0) SPCUDA(run_bfs(0, a, st));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, t->row_off, u.n + 1, st);
  Scratch<unsigned char> tmp;
  SPCUDA(tmp.alloc(tb + 16, st));
  SPCUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, t->row_off, u.n + 1, st));
  SPCUDA(cudaMemcpyAsync(&t->total, t->row_off + u.n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaStreamSynchronize(st));
  SPCUDA(cudaMallocAsync(&t->cols, sizeof(int32_t) * (t->total ? t->total : 1), st));
  SPCUDA(cudaMallocAsync(&t->dist, sizeof(uint16_t) * (t->total ? t->total : 1), st));
  a.out_off = t->row_off;
  a.out_cols = t->cols;
  a.out_dist = t->dist;
  if (u.n > 0) SPCUDA(run_bfs(1, a, st));
  SPCUDA(cudaStreamSynchronize(st));
  return GTE_OK;
}

// ---------------------------------------------------------------- pair distances
__device__ __forceinline__ int ball_find(const int64_t* off, const int32_t* cols, int32_t i, int32_t j) {
  int64_t lo = off[i], hi = off[i + 1];
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    if (cols[mid] < j) lo = mid + 1; else hi = mid;
  }
  return (lo < off[i + 1] && cols[lo] == j) ? (int)lo : -1;
}

// warp per pair: d <= 2 from B2(i); else min over B2(i) ∩ B2(j) of d_i + d_j
// (3 or 4); else -1 (>= 5) unless cap <= 4 (then cap + 1)
__global__ void pairs_kernel(int64_t np, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                             const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                             const uint16_t* __restrict__ dist, int32_t cap, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = wid; p < np; p += nw) {
    const int32_t i = src[p], j = dst[p];
    const int at = ball_find(off, cols, i, j);
    if (at >= 0) {
      if (lane == 0) out[p] = dist[at];
      continue;
    }
    if (cap <= 2) {
      if (lane == 0) out[p] = cap + 1;
      continue;
    }
    // meet in the middle: scan the smaller ball, search the larger
    int32_t a = i, b = j;
    if (off[i + 1] - off[i] > off[j + 1] - off[j]) {
      a = j;
      b = i;
    }
    int best = 1 << 20;
    for (int64_t x = off[a] + lane; x < off[a + 1]; x += 32) {
      const int y = ball_find(off, cols, b, cols[x]);
      if (y >= 0) best = min(best, (int)dist[x] + (int)dist[y]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) out[p] = best <= 4 ? (best <= cap ? best : cap + 1) : (cap <= 4 ? cap + 1 : -1);
  }
}

int spd_pairs_impl(cudaStream_t st, const UAdj& u, int32_t cap, int64_t np, const int32_t* d_src,
                   const int32_t* d_dst, int32_t* d_out) {
  if (np == 0) return GTE_OK;
  gte_spd b2;
  int rc = build_table(st, u, std::min(cap, 2), &b2);
  struct Free {
    gte_spd& t;
    cudaStream_t st;
    ~Free() {
      cudaFreeAsync(t.row_off, st);
      cudaFreeAsync(t.cols, st);
      cudaFreeAsync(t.dist, st);
    }
  } fr{b2, st};
  if (rc) return rc;
  const int64_t blocks = std::min<int64_t>((np * 32 + 255) / 256, 148 * 64);
  pairs_kernel<<<(unsigned)blocks, 256, 0, st>>>(np, d_src, d_dst, b2.row_off, b2.cols, b2.dist, cap, d_out);
  SPCUDA(cudaGetLastError());
  if (cap <= 4) return GTE_OK;
  // the rest (d >= 5): early-exit BFS per distinct source
  std::vector<int32_t> out(np), hs(np), hd(np);
  SPCUDA(cudaMemcpyAsync(out.data(), d_out, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaMemcpyAsync(hs.data(), d_src, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaMemcpyAsync(hd.data(), d_dst, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> left;
  for (int64_t p = 0; p < np; ++p)
    if (out[p] < 0) left.push_back(p);
  if (left.empty()) return GTE_OK;
  std::stable_sort(left.begin(), left.end(), [&](int64_t x, int64_t y) { return hs[x] < hs[y]; });
  std::vector<int32_t> srcs, toff{0}, tgt;
  for (size_t k = 0; k < left.size(); ++k) {
    if (k == 0 || hs[left[k]] != hs[left[k - 1]]) {
      if (k) toff.push_back((int32_t)tgt.size());
      srcs.push_back(hs[left[k]]);
    }
    tgt.push_back(hd[left[k]]);
  }
  toff.push_back((int32_t)tgt.size());
  Scratch<int32_t> d_srcs, d_toff, d_tgt, d_td;
  SPCUDA(d_srcs.alloc(srcs.size(), st));
  SPCUDA(d_toff.alloc(toff.size(), st));
  SPCUDA(d_tgt.alloc(tgt.size(), st));
  SPCUDA(d_td.alloc(tgt.size(), st));
  SPCUDA(cudaMemcpyAsync(d_srcs.p, srcs.data(), 4 * srcs.size(), cudaMemcpyHostToDevice, st));
  SPCUDA(cudaMemcpyAsync(d_toff.p, toff.data(), 4 * toff.size(), cudaMemcpyHostToDevice, st));
  SPCUDA(cudaMemcpyAsync(d_tgt.p, tgt.data(), 4 * tgt.size(), cudaMemcpyHostToDevice, st));
  SPCUDA(cudaMemsetAsync(d_td.p, 0xff, 4 * tgt.size(), st));
  BfsArgs a;
  a.n = u.n;
  a.cap = cap;
  a.off = u.off.p;
  a.adj = u.adj.p;
  a.srcs = d_srcs.p;
  a.nsrc = (int32_t)srcs.size();
  a.tgt_off = d_toff.p;
  a.tgt = d_tgt.p;
  a.tgt_dist = d_td.p;
  SPCUDA(run_bfs(2, a, st));
  std::vector<int32_t> td(tgt.size());
  SPCUDA(cudaMemcpyAsync(td.data(), d_td.p, 4 * td.size(), cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaStreamSynchronize(st));
  for (size_t k = 0; k < left.size(); ++k) out[left[k]] = td[k] < 0 ? cap + 1 : td[k];
  SPCUDA(cudaMemcpyAsync(d_out, out.data(), sizeof(int32_t) * np, cudaMemcpyHostToDevice, st));
  SPCUDA(cudaStreamSynchronize(st));
  return GTE_OK;
}

// pattern pair -> (original i, j) and the Trainer's fixed buckets
__global__ void pattern_pairs_kernel(int32_t rows, int32_t nnz, const int32_t* __restrict__ rp,
                                     const int32_t* __restrict__ cols, const int64_t* __restrict__ inv, int64_t global,
                                     int64_t graph_n, int32_t unreachable, int32_t* __restrict__ bucket,
                                     int32_t* __restrict__ pi, int32_t* __restrict__ pj, int32_t* __restrict__ need) {
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const int64_t i = inv[r];
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int64_t j = inv[cols[e]];
      int32_t b = -1;
      if (i == j) b = 0;
      else if (i == global || j == global) b = 1;
      else if (i >= graph_n || j >= graph_n) b = unreachable;
      bucket[e] = b;
      pi[e] = (int32_t)i;
      pj[e] = (int32_t)j;
      need[e] = b < 0 ? 1 : 0;
    }
  }
}

}  // namespace

extern "C" {

int gte_spd_table(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                  int64_t max_dist, gte_spd** out) {
  if (max_dist < 0) return set_error(GTE_CONFIG, "spd_table: max_dist must be >= 0");  // graph.cpp:217
  if (max_dist > 255) return set_error(GTE_CONFIG, "spd_table: max_dist must be <= 255");
  if (n >= (1ll << 31) || nnz >= (1ll << 30)) return set_error(GTE_CONFIG, "spd_table: graph exceeds int32 indices");
  cudaStream_t st = static_cast<cudaStream_t>(ctx_stream(c));
  UAdj u;
  SPCUDA(build_uadj(st, (int32_t)n, (int32_t)nnz, d_row_ptr, d_cols, u));
  auto* t = new gte_spd();
  int rc = build_table(st, u, (int32_t)max_dist, t);
  ctx_launch_counter(c) += 4;
  if (rc) {
    gte_spd_destroy(t);
    return rc;
  }
  *out = t;
  return GTE_OK;
}

int gte_spd_info(const gte_spd* t, int64_t* n, int64_t* max_dist, int64_t* total) {
  if (n) *n = t->n;
  if (max_dist) *max_dist = t->max_dist;
  if (total) *total = t->total;
  return GTE_OK;
}

int gte_spd_copy_host(const gte_spd* t, int64_t* row_off, int64_t* cols, uint16_t* dist) {
  std::vector<int32_t> c32(t->total);
  SPCUDA(cudaMemcpy(row_off, t->row_off, sizeof(int64_t) * (t->n + 1), cudaMemcpyDeviceToHost));
  if (t->total) {
    SPCUDA(cudaMemcpy(c32.data(), t->cols, sizeof(int32_t) * t->total, cudaMemcpyDeviceToHost));
    SPCUDA(cudaMemcpy(dist, t->dist, sizeof(uint16_t) * t->total, cudaMemcpyDeviceToHost));
  }
  for (int64_t x = 0; x < t->total; ++x) cols[x] = c32[x];
  return GTE_OK;
}

int gte_spd_destroy(gte_spd* t) {
  if (!t) return GTE_OK;
  cudaFree(t->row_off);
  cudaFree(t->cols);
  cudaFree(t->dist);
  delete t;
  return GTE_OK;
}

int gte_spd_pairs(gte_ctx* c, int64_t n, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                  int64_t max_dist, int64_t n_pairs, const int32_t* d_src, const int32_t* d_dst, int32_t* d_dist) {
  if (max_dist < 0) return set_error(GTE_CONFIG, "spd_table: max_dist must be >= 0");
  if (max_dist > 255) return set_error(GTE_CONFIG, "spd_table: max_dist must be <= 255");
  cudaStream_t st = static_cast<cudaStream_t>(ctx_stream(c));
  UAdj u;
  SPCUDA(build_uadj(st, (int32_t)n, (int32_t)nnz, d_row_ptr, d_cols, u));
  ctx_launch_counter(c) += 6;
  return spd_pairs_impl(st, u, (int32_t)max_dist, n_pairs, d_src, d_dst, d_dist);
}

int gte_pattern_buckets_graph(gte_ctx* c, int64_t rows, int64_t nnz, const int32_t* d_row_ptr, const int32_t* d_cols,
                              const int64_t* d_perm_inverse, int64_t global_index, int64_t graph_n,
                              int64_t graph_nnz, const int32_t* d_graph_row_ptr, const int32_t* d_graph_cols,
                              int64_t max_dist, int32_t* d_buckets) {
  if (max_dist < 0) return set_error(GTE_CONFIG, "spd_table: max_dist must be >= 0");
  cudaStream_t st = static_cast<cudaStream_t>(ctx_stream(c));
  Scratch<int32_t> pi, pj, need, pos, ci, cj, cd;
  SPCUDA(pi.alloc(nnz, st));
  SPCUDA(pj.alloc(nnz, st));
  SPCUDA(need.alloc(nnz + 1, st));
  if (rows > 0)
    pattern_pairs_kernel<<<(unsigned)std::min<int64_t>((rows + 255) / 256, 148 * 16), 256, 0, st>>>(
        (int32_t)rows, (int32_t)nnz, d_row_ptr, d_cols, d_perm_inverse, global_index, graph_n, (int32_t)max_dist + 1,
        d_buckets, pi.p, pj.p, need.p);
  SPCUDA(cudaGetLastError());
  // compact the pairs that need a distance, resolve, scatter back
  std::vector<int32_t> hn(nnz), hi(nnz), hj(nnz);
  SPCUDA(cudaMemcpyAsync(hn.data(), need.p, 4 * nnz, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaMemcpyAsync(hi.data(), pi.p, 4 * nnz, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaMemcpyAsync(hj.data(), pj.p, 4 * nnz, cudaMemcpyDeviceToHost, st));
  SPCUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> idx, si, sj;
  for (int64_t e = 0; e < nnz; ++e)
    if (hn[e]) {
      idx.push_back((int32_t)e);
      si.push_back(hi[e]);
      sj.push_back(hj[e]);
    }
  const int64_t np = (int64_t)idx.size();
  if (np) {
    SPCUDA(ci.alloc(np, st));
    SPCUDA(cj.alloc(np, st));
    SPCUDA(cd.alloc(np, st));
    SPCUDA(cudaMemcpyAsync(ci.p, si.data(), 4 * np, cudaMemcpyHostToDevice, st));
    SPCUDA(cudaMemcpyAsync(cj.p, sj.data(), 4 * np, cudaMemcpyHostToDevice, st));
    UAdj u;
    SPCUDA(build_uadj(st, (int32_t)graph_n, (int32_t)graph_nnz, d_graph_row_ptr, d_graph_cols, u));
    int rc = spd_pairs_impl(st, u, (int32_t)max_dist, np, ci.p, cj.p, cd.p);
    if (rc) return rc;
    std::vector<int32_t> hd(np), hb(nnz);
    SPCUDA(cudaMemcpyAsync(hd.data(), cd.p, 4 * np, cudaMemcpyDeviceToHost, st));
    SPCUDA(cudaMemcpyAsync(hb.data(), d_buckets, 4 * nnz, cudaMemcpyDeviceToHost, st));
    SPCUDA(cudaStreamSynchronize(st));
    for (int64_t k = 0; k < np; ++k) hb[idx[k]] = hd[k];
    SPCUDA(cudaMemcpyAsync(d_buckets, hb.data(), 4 * nnz, cudaMemcpyHostToDevice, st));
  }
  SPCUDA(cudaStreamSynchronize(st));
  ctx_launch_counter(c) += 2;
  return GTE_OK;
}

// Dense-epoch bucket matrix (model.cpp:395-423 with dense_pattern_exec):
// out[r][c] for execution rows r < s_real and real columns c < s_real; pad
// rows/columns are left unset (pad rows attend only themselves, unbiased).
int gte_dense_buckets(gte_ctx* c, int64_t S, int64_t s_real, const int64_t* d_perm_forward,
                      const int64_t* d_perm_inverse, int64_t global_index, int64_t graph_n, int64_t graph_nnz,
                      const int32_t* d_graph_row_ptr, const int32_t* d_graph_cols, int64_t max_dist, uint8_t* d_out) {
  if (max_dist < 0) return set_error(GTE_CONFIG, "spd_table: max_dist must be >= 0");
  if (max_dist > 253) return set_error(GTE_CONFIG, "dense buckets: max_dist must be <= 253");
  if (s_real < 0 || s_real > S || graph_n > s_real) return set_error(GTE_CONFIG, "dense buckets: bad sizes");
  cudaStream_t st = static_cast<cudaStream_t>(ctx_stream(c));
  UAdj u;
  SPCUDA(build_uadj(st, (int32_t)graph_n, (int32_t)graph_nnz, d_graph_row_ptr, d_graph_cols, u));
  BfsArgs a;
  a.n = (int32_t)graph_n;
  a.cap = (int32_t)max_dist;
  a.off = u.off.p;
  a.adj = u.adj.p;
  a.nsrc = (int32_t)s_real;
  a.inv = d_perm_inverse;
  a.fwd = d_perm_forward;
  a.S = S;
  a.s_real = s_real;
  a.global = global_index;
  a.graph_n = (int32_t)graph_n;
  a.rows_out = d_out;
  if (s_real > 0) SPCUDA(run_bfs(3, a, st));
  SPCUDA(cudaStreamSynchronize(st));
  ctx_launch_counter(c) += 5;
  return GTE_OK;
}

}  // extern "C"

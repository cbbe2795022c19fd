// Device graph transforms of the cluster-aware reorder (bisection.h):
// segmented sort / run-length / reduce-by-key / scan over the arc list of one
// level, instead of the reference's per-node host loops
// (proj/src/partition.cpp:40-66 ugraph_from, :73-109 contract, :352-391 the
// subgraphs of a bisection). Every result is ordered exactly as the
// reference orders it (coarse ids by first member, neighbours ascending,
// subgraph ids in parent order), so the host's greedy passes see the same
// graphs.
#include <cub/cub.cuh>

#include <stdexcept>
#include <string>

#include "bisection.h"

namespace gte_b200 {
namespace part {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("reorder (device ") + what + "): " + cudaGetErrorString(e));
}

// stream-ordered scratch that frees itself
template <typename T>
struct DBuf {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  DBuf(size_t n, cudaStream_t s) : st(s) { ck(cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), s), "alloc"); }
  ~DBuf() { cudaFreeAsync(p, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

constexpr uint64_t kNone = ~0ull;  // sorts after every real (u, v) key
inline unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

template <typename X>
void up(X* d, const X* h, size_t n, cudaStream_t st) {
  if (n) ck(cudaMemcpyAsync(d, h, sizeof(X) * n, cudaMemcpyHostToDevice, st), "upload");
}
template <typename X>
void down(X* h, const X* d, size_t n, cudaStream_t st) {
  if (n) ck(cudaMemcpyAsync(h, d, sizeof(X) * n, cudaMemcpyDeviceToHost, st), "download");
}

// owner row of every arc: rows scatter their index over their arc range
__global__ void arc_owner_kernel(const int64_t* __restrict__ off, int64_t n, int32_t* __restrict__ owner) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  for (int64_t a = off[u]; a < off[u + 1]; ++a) owner[a] = (int32_t)u;
}

// directed arc (u, v) -> keys (u, v) and (v, u); self arcs -> kNone
__global__ void both_ways_kernel(const int32_t* __restrict__ owner, const int64_t* __restrict__ cols, int64_t m,
                                 uint64_t* __restrict__ keys) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const uint64_t u = (uint64_t)owner[a], v = (uint64_t)cols[a];
  keys[2 * a] = u == v ? kNone : (u << 32 | v);
  keys[2 * a + 1] = u == v ? kNone : (v << 32 | u);
}

// unique (u, v) keys -> heads, per-row arc counts
__global__ void decode_kernel(const uint64_t* __restrict__ keys, int64_t r, int32_t* __restrict__ head,
                              int64_t* __restrict__ deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  const uint64_t k = keys[i];
  head[i] = (int32_t)(k & 0xffffffffu);
  atomicAdd(reinterpret_cast<unsigned long long*>(deg + (k >> 32)), 1ull);
}

__global__ void first_flag_kernel(const int32_t* __restrict__ mate, int64_t n, int32_t* __restrict__ flag) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n) flag[u] = mate[u] >= (int32_t)u ? 1 : 0;
}

__global__ void cmap_kernel(const int32_t* __restrict__ mate, const int32_t* __restrict__ flag,
                            const int32_t* __restrict__ rank, const int32_t* __restrict__ vw, int64_t n,
                            int32_t* __restrict__ cmap, int32_t* __restrict__ cvw) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int32_t c = flag[u] ? rank[u] : rank[mate[u]];
  cmap[u] = c;
  atomicAdd(cvw + c, vw[u]);
}

// arc (u, v, w) -> key (cmap u, cmap v), value w; arcs inside a coarse node -> kNone
__global__ void coarse_arc_kernel(const int32_t* __restrict__ owner, const int32_t* __restrict__ nbr,
                                  const int32_t* __restrict__ cmap, int64_t m, uint64_t* __restrict__ keys) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const uint64_t cu = (uint64_t)cmap[owner[a]], cv = (uint64_t)cmap[nbr[a]];
  keys[a] = cu == cv ? kNone : (cu << 32 | cv);
}

// per side: local id = rank among that side's nodes; arc kept iff both ends on the side
__global__ void side_flag_kernel(const uint8_t* __restrict__ side, int64_t n, int32_t* __restrict__ is1) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n) is1[u] = side[u] ? 1 : 0;
}

__global__ void keep_kernel(const int32_t* __restrict__ owner, const int32_t* __restrict__ nbr,
                            const uint8_t* __restrict__ side, int64_t m, int32_t* __restrict__ keep0,
                            int32_t* __restrict__ keep1) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const uint8_t su = side[owner[a]], sv = side[nbr[a]];
  keep0[a] = (su == 0 && sv == 0) ? 1 : 0;
  keep1[a] = (su == 1 && sv == 1) ? 1 : 0;
}

__global__ void split_scatter_kernel(const int32_t* __restrict__ owner, const int32_t* __restrict__ nbr,
                                     const int32_t* __restrict__ wt, const uint8_t* __restrict__ side,
                                     const int32_t* __restrict__ rank1, const int32_t* __restrict__ pos0,
                                     const int32_t* __restrict__ pos1, int64_t m, int32_t* __restrict__ adj0,
                                     int32_t* __restrict__ w0, int32_t* __restrict__ adj1, int32_t* __restrict__ w1) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  const int32_t u = owner[a], v = nbr[a];
  const uint8_t s = side[u];
  if (side[v] != s) return;
  const int32_t lv = s ? rank1[v] : v - rank1[v];  // rank among side-s nodes
  if (s) {
    adj1[pos1[a]] = lv;
    w1[pos1[a]] = wt[a];
  } else {
    adj0[pos0[a]] = lv;
    w0[pos0[a]] = wt[a];
  }
}

__global__ void split_rows_kernel(const int64_t* __restrict__ off, const uint8_t* __restrict__ side,
                                  const int32_t* __restrict__ rank1, const int32_t* __restrict__ pos0,
                                  const int32_t* __restrict__ pos1, int64_t n, int64_t* __restrict__ off0,
                                  int64_t* __restrict__ off1, int32_t* __restrict__ ids0, int32_t* __restrict__ ids1) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  if (side[u]) {
    off1[rank1[u]] = pos1[off[u]];
    ids1[rank1[u]] = (int32_t)u;
  } else {
    off0[u - rank1[u]] = pos0[off[u]];
    ids0[u - rank1[u]] = (int32_t)u;
  }
}

template <typename F>
void cub_call(cudaStream_t st, F&& f) {  // f(tmp, bytes): size query, then run
  size_t bytes = 0;
  ck(f(nullptr, bytes), "cub size");
  DBuf<unsigned char> tmp(bytes + 16, st);
  ck(f(tmp.p, bytes), "cub");
}

}  // namespace

void dev_symmetrize(cudaStream_t st, int64_t n, const int64_t* row_off, const int64_t* cols, WGraph& out) {
  const int64_t m = row_off[n];
  out.n = n;
  out.vw.assign(n, 1);
  out.xoff.assign(n + 1, 0);
  out.nbr.clear();
  out.wt.clear();
  if (m == 0) return;
  DBuf<int64_t> off(n + 1, st), col(m, st);
  up(off.p, row_off, n + 1, st);
  up(col.p, cols, m, st);
  DBuf<int32_t> owner(m, st);
  arc_owner_kernel<<<blocks_for(n), 256, 0, st>>>(off.p, n, owner.p);
  DBuf<uint64_t> keys(2 * m, st), sorted(2 * m, st), uniq(2 * m, st);
  both_ways_kernel<<<blocks_for(m), 256, 0, st>>>(owner.p, col.p, m, keys.p);
  const int items = (int)(2 * m);
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceRadixSort::SortKeys(t, b, keys.p, sorted.p, items, 0, 64, st); });
  DBuf<int32_t> counts(2 * m, st), nruns(1, st);
  cub_call(st, [&](void* t, size_t& b) {
    return cub::DeviceRunLengthEncode::Encode(t, b, sorted.p, uniq.p, counts.p, nruns.p, items, st);
  });
  int32_t r = 0;
  uint64_t last = 0;
  down(&r, nruns.p, 1, st);
  ck(cudaStreamSynchronize(st), "sync");
  if (r > 0) {
    down(&last, uniq.p + (r - 1), 1, st);
    ck(cudaStreamSynchronize(st), "sync");
    if (last == kNone) --r;  // the self arcs' run
  }
  DBuf<int32_t> head(r, st);
  DBuf<int64_t> deg(n + 1, st);
  ck(cudaMemsetAsync(deg.p, 0, sizeof(int64_t) * (n + 1), st), "memset");
  if (r > 0) decode_kernel<<<blocks_for(r), 256, 0, st>>>(uniq.p, r, head.p, deg.p);
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, deg.p, off.p, (int)(n + 1), st); });
  out.nbr.resize(r);
  out.wt.resize(r);
  down(out.nbr.data(), head.p, r, st);
  down(out.wt.data(), counts.p, r, st);
  down(out.xoff.data(), off.p, n + 1, st);
  ck(cudaStreamSynchronize(st), "sync");
}

void dev_contract(cudaStream_t st, const WGraph& g, const std::vector<int32_t>& mate, WGraph& coarse,
                  std::vector<int32_t>& cmap) {
  const int64_t n = g.n, m = g.arcs();
  DBuf<int64_t> off(n + 1, st);
  DBuf<int32_t> nbr(m, st), wt(m, st), vw(n, st), dm(n, st), flag(n, st), rank(n, st), cm(n, st), owner(m, st);
  up(off.p, g.xoff.data(), n + 1, st);
  up(nbr.p, g.nbr.data(), m, st);
  up(wt.p, g.wt.data(), m, st);
  up(vw.p, g.vw.data(), n, st);
  up(dm.p, mate.data(), n, st);
  first_flag_kernel<<<blocks_for(n), 256, 0, st>>>(dm.p, n, flag.p);
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, flag.p, rank.p, (int)n, st); });
  int32_t last_rank = 0, last_flag = 0;
  down(&last_rank, rank.p + (n - 1), 1, st);
  down(&last_flag, flag.p + (n - 1), 1, st);
  ck(cudaStreamSynchronize(st), "sync");
  const int64_t nc = (int64_t)last_rank + last_flag;
  DBuf<int32_t> cvw(nc, st);
  ck(cudaMemsetAsync(cvw.p, 0, sizeof(int32_t) * (nc ? nc : 1), st), "memset");
  cmap_kernel<<<blocks_for(n), 256, 0, st>>>(dm.p, flag.p, rank.p, vw.p, n, cm.p, cvw.p);
  coarse.n = nc;
  coarse.vw.resize(nc);
  coarse.xoff.assign(nc + 1, 0);
  cmap.resize(n);
  down(cmap.data(), cm.p, n, st);
  down(coarse.vw.data(), cvw.p, nc, st);
  if (m == 0) {
    coarse.nbr.clear();
    coarse.wt.clear();
    ck(cudaStreamSynchronize(st), "sync");
    return;
  }
  arc_owner_kernel<<<blocks_for(n), 256, 0, st>>>(off.p, n, owner.p);
  DBuf<uint64_t> keys(m, st), skeys(m, st), ukeys(m, st);
  DBuf<int32_t> swt(m, st), sums(m, st), nruns(1, st);
  coarse_arc_kernel<<<blocks_for(m), 256, 0, st>>>(owner.p, nbr.p, cm.p, m, keys.p);
  const int items = (int)m;
  cub_call(st, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, keys.p, skeys.p, wt.p, swt.p, items, 0, 64, st);
  });
  cub_call(st, [&](void* t, size_t& b) {
    return cub::DeviceReduce::ReduceByKey(t, b, skeys.p, ukeys.p, swt.p, sums.p, nruns.p, cub::Sum(), items, st);
  });
  int32_t r = 0;
  uint64_t last = 0;
  down(&r, nruns.p, 1, st);
  ck(cudaStreamSynchronize(st), "sync");
  if (r > 0) {
    down(&last, ukeys.p + (r - 1), 1, st);
    ck(cudaStreamSynchronize(st), "sync");
    if (last == kNone) --r;  // the arcs inside coarse nodes
  }
  DBuf<int32_t> head(r, st);
  DBuf<int64_t> deg(nc + 1, st), coff(nc + 1, st);
  ck(cudaMemsetAsync(deg.p, 0, sizeof(int64_t) * (nc + 1), st), "memset");
  if (r > 0) decode_kernel<<<blocks_for(r), 256, 0, st>>>(ukeys.p, r, head.p, deg.p);
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, deg.p, coff.p, (int)(nc + 1), st); });
  coarse.nbr.resize(r);
  coarse.wt.resize(r);
  down(coarse.nbr.data(), head.p, r, st);
  down(coarse.wt.data(), sums.p, r, st);
  down(coarse.xoff.data(), coff.p, nc + 1, st);
  ck(cudaStreamSynchronize(st), "sync");
}

void dev_split(cudaStream_t st, const WGraph& g, const std::vector<uint8_t>& side, WGraph (&sub)[2],
               std::vector<int32_t> (&ids)[2]) {
  const int64_t n = g.n, m = g.arcs();
  DBuf<int64_t> off(n + 1, st);
  DBuf<int32_t> nbr(m, st), wt(m, st), is1(n, st), rank1(n, st), owner(m, st);
  DBuf<uint8_t> sd(n, st);
  up(off.p, g.xoff.data(), n + 1, st);
  up(nbr.p, g.nbr.data(), m, st);
  up(wt.p, g.wt.data(), m, st);
  up(sd.p, side.data(), n, st);
  side_flag_kernel<<<blocks_for(n), 256, 0, st>>>(sd.p, n, is1.p);
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, is1.p, rank1.p, (int)n, st); });
  int64_t n1 = 0;
  for (uint8_t s : side) n1 += s ? 1 : 0;
  const int64_t ns[2] = {n - n1, n1};
  // arc positions inside each side's arc list (one extra slot: the total)
  DBuf<int32_t> keep0(m + 1, st), keep1(m + 1, st), pos0(m + 1, st), pos1(m + 1, st);
  ck(cudaMemsetAsync(keep0.p + m, 0, sizeof(int32_t), st), "memset");
  ck(cudaMemsetAsync(keep1.p + m, 0, sizeof(int32_t), st), "memset");
  if (m > 0) {
    arc_owner_kernel<<<blocks_for(n), 256, 0, st>>>(off.p, n, owner.p);
    keep_kernel<<<blocks_for(m), 256, 0, st>>>(owner.p, nbr.p, sd.p, m, keep0.p, keep1.p);
  }
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, keep0.p, pos0.p, (int)(m + 1), st); });
  cub_call(st, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, keep1.p, pos1.p, (int)(m + 1), st); });
  int32_t tot[2] = {0, 0};
  down(&tot[0], pos0.p + m, 1, st);
  down(&tot[1], pos1.p + m, 1, st);
  ck(cudaStreamSynchronize(st), "sync");
  DBuf<int32_t> adj0(tot[0], st), w0(tot[0], st), adj1(tot[1], st), w1(tot[1], st), i0(ns[0], st), i1(ns[1], st);
  DBuf<int64_t> off0(ns[0] + 1, st), off1(ns[1] + 1, st);
  if (m > 0)
    split_scatter_kernel<<<blocks_for(m), 256, 0, st>>>(owner.p, nbr.p, wt.p, sd.p, rank1.p, pos0.p, pos1.p, m, adj0.p,
                                                         w0.p, adj1.p, w1.p);
  split_rows_kernel<<<blocks_for(n), 256, 0, st>>>(off.p, sd.p, rank1.p, pos0.p, pos1.p, n, off0.p, off1.p, i0.p, i1.p);
  int32_t* adjs[2] = {adj0.p, adj1.p};
  int32_t* ws[2] = {w0.p, w1.p};
  int64_t* offs[2] = {off0.p, off1.p};
  int32_t* idp[2] = {i0.p, i1.p};
  for (int s = 0; s < 2; ++s) {
    WGraph& h = sub[s];
    h.n = ns[s];
    h.xoff.assign(ns[s] + 1, tot[s]);
    h.nbr.resize(tot[s]);
    h.wt.resize(tot[s]);
    ids[s].resize(ns[s]);
    down(h.xoff.data(), offs[s], ns[s], st);  // last entry = total (set above)
    down(h.nbr.data(), adjs[s], tot[s], st);
    down(h.wt.data(), ws[s], tot[s], st);
    down(ids[s].data(), idp[s], ns[s], st);
  }
  ck(cudaStreamSynchronize(st), "sync");
  for (int s = 0; s < 2; ++s) {
    sub[s].vw.resize(ns[s]);
    for (int64_t i = 0; i < ns[s]; ++i) sub[s].vw[i] = g.vw[ids[s][i]];
  }
}

}  // namespace part
}  // namespace gte_b200

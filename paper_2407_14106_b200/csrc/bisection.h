// Cluster-aware node reordering (reference proj/src/partition.cpp:15-433):
// multilevel recursive bisection. The data-parallel graph transforms run on
// the GPU (partition_gpu.cu: symmetrise, contract a matching, split along a
// bisection); the greedy decisions whose order the reference fixes run on the
// host (bisection.cpp: matching, BFS seeds, region growth, FM refinement,
// exact rebalance) with heap-selected moves instead of the reference's
// O(n) scans, so the permutation is bit-identical at any size.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace gte_b200 {
namespace part {

// Weighted undirected graph (both arc directions stored), neighbour lists
// ascending, no self arcs. Host mirror of one level of the hierarchy.
struct WGraph {
  int64_t n = 0;
  std::vector<int64_t> xoff{0};  // [n + 1]
  std::vector<int32_t> nbr;      // arc heads
  std::vector<int32_t> wt;       // arc weights (multiplicities, summed when contracted)
  std::vector<int32_t> vw;       // node weights (fine nodes merged)
  int64_t arcs() const { return xoff[n]; }
};

// ---- device transforms (partition_gpu.cu); throw std::runtime_error ----
// directed CSR -> WGraph: u != v arcs in both directions, weight = how many
// arcs join u and v (partition.cpp:40-66)
void dev_symmetrize(cudaStream_t st, int64_t n, const int64_t* row_off, const int64_t* cols, WGraph& out);
// coarse node of u = rank of min(u, mate[u]) among such; coarse arcs summed,
// internal arcs dropped (partition.cpp:73-109). cmap[u] = coarse node of u.
void dev_contract(cudaStream_t st, const WGraph& g, const std::vector<int32_t>& mate, WGraph& coarse,
                  std::vector<int32_t>& cmap);
// the two sides' induced subgraphs, nodes renumbered in increasing order
// (partition.cpp:352-391); ids[s] = parent node of each local node
void dev_split(cudaStream_t st, const WGraph& g, const std::vector<uint8_t>& side, WGraph (&sub)[2],
               std::vector<int32_t> (&ids)[2]);

}  // namespace part

// Bit-identical to the reference gte::reorder (partition.cpp:413-433);
// caller validates k (power of two, 1 <= k <= n). Needs a CUDA device.
void reorder_cluster(int64_t n, const int64_t* row_off, const int64_t* cols, int64_t k, uint64_t seed,
                     int64_t* forward, int64_t* inverse);

}  // namespace gte_b200

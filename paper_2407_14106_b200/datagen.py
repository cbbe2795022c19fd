"""Synthetic graph generators for the benchmark configs.

Host-side tooling, not part of the attention hot path. ``c1_graph`` reproduces
the C1 recipe draw for draw (mt19937_64 + libstdc++ uniform_int_distribution);
``community_graph`` is the O(E) community-structured generator used for the
products-shaped C3 sequence (planted communities, mostly intra-community arcs,
lognormal out-degree), with node ids shuffled so the reorder has real work.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (standardised), pure Python — fine for ~1e5 draws."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _M64
        for i in range(1, 312):
            p = mt[i - 1]
            mt[i] = (6364136223846793005 * (p ^ (p >> 62)) + i) & _M64
        self.mt = mt
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            v = mt[(i + 156) % 312] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        z = self.mt[self.idx]
        self.idx += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000
        z ^= (z << 37) & 0xFFF7EEE000000000
        z ^= z >> 43
        return z & _M64

    def uniform_int(self, a: int, b: int) -> int:
        """std::uniform_int_distribution<int64_t>(a, b) (libstdc++ Lemire path)."""
        rng = (b - a) + 1
        prod = self() * rng
        low = prod & _M64
        if low < rng:
            thr = ((1 << 64) - rng) % rng
            while low < thr:
                prod = self() * rng
                low = prod & _M64
        return a + (prod >> 64)


def c1_edges(n: int = 4096, draws: int = 16, seed: int = 1):
    """C1 recipe: per node `draws` v ~ U[0, n) from mt19937_64(seed), v == u dropped."""
    g = MT19937_64(seed)
    src, dst = [], []
    for u in range(n):
        for _ in range(draws):
            v = g.uniform_int(0, n - 1)
            if v != u:
                src.append(u)
                dst.append(v)
    return np.array(src, dtype=np.int64), np.array(dst, dtype=np.int64)


def csr_from_pairs(n: int, src: np.ndarray, dst: np.ndarray, self_loops: bool = True):
    """Canonical CSR (sorted, unique) of a pair list, optionally with every
    diagonal pair added — numerically what graph_from_edges + add_self_loops
    produce (reference proj/src/graph.cpp:49-66, 127-149)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if self_loops:
        ar = np.arange(n, dtype=np.int64)
        src = np.concatenate([src, ar])
        dst = np.concatenate([dst, ar])
    key = np.unique(src * n + dst)
    rows = key // n
    cols = key % n
    row_off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_off, rows + 1, 1)
    np.cumsum(row_off, out=row_off)
    return row_off, cols.astype(np.int64)


def community_graph(n: int, arcs_per_node: float, community: int = 256, intra: float = 0.8,
                    sigma: float = 1.0, seed: int = 7, shuffle: bool = True):
    """Products-shaped synthetic sequence: n nodes in
    planted communities of `community`, lognormal out-degree with mean
    `arcs_per_node`, `intra` of arcs inside the community; node ids shuffled.
    Returns (row_off, cols) int64 with self-loops, sorted and unique."""
    rs = np.random.default_rng(seed)
    mu = np.log(arcs_per_node) - 0.5 * sigma * sigma
    deg = np.maximum(1, np.round(rs.lognormal(mu, sigma, size=n))).astype(np.int64)
    deg = np.minimum(deg, n - 1)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    m = src.shape[0]
    comm = src // community
    inside = rs.random(m) < intra
    dst = np.where(inside, comm * community + rs.integers(0, community, size=m), rs.integers(0, n, size=m))
    dst = np.minimum(dst, n - 1)
    keep = dst != src
    src, dst = src[keep], dst[keep]
    if shuffle:
        relabel = rs.permutation(n).astype(np.int64)
        src, dst = relabel[src], relabel[dst]
    return csr_from_pairs(n, src, dst, self_loops=True)


def products_c3(seed: int = 7):
    """C3: S = 262,144, ~25.26 arcs/node -> E ~ 6.8M incl. loops."""
    return community_graph(262144, 61859140 / 2449029, community=256, intra=0.8, sigma=1.0, seed=seed)


def arxiv_c2(seed: int = 11, n: int = 169343, arcs: int = 1166243):
    """C2 (ogbn-arxiv shape): n = 169,343 nodes with exactly
    `arcs` distinct non-loop arcs (uniform endpoints, oversampled then cut),
    plus every self-loop -> E = 1,335,586. Returns (row_off, cols) int64."""
    rs = np.random.default_rng(seed)
    keys = np.empty(0, dtype=np.int64)
    while keys.shape[0] < arcs:
        m = int(1.1 * (arcs - keys.shape[0])) + 1024
        s = rs.integers(0, n, m, dtype=np.int64)
        t = rs.integers(0, n, m, dtype=np.int64)
        k = s[s != t] * n + t[s != t]
        keys = np.unique(np.concatenate([keys, k]))
    keys = rs.permutation(keys)[:arcs]
    return csr_from_pairs(n, keys // n, keys % n)


def malnet_c4(seed: int = 13, n: int = 524288, arcs_per_node: float = 35167 / 15378):
    """C4 (MalNet shape): n = 524,288 graph nodes at 2.29
    arcs/node plus one global token (index n) attending to and attended by
    every node (proj/src/model.cpp:349-357), self-loops added ->
    E ~ 2.77M. Returns (row_off, cols) int64 over n + 1 rows."""
    ro, co = community_graph(n, arcs_per_node, community=256, intra=0.8, sigma=1.0, seed=seed)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    nodes = np.arange(n, dtype=np.int64)
    glob = np.full(n, n, dtype=np.int64)
    return csr_from_pairs(n + 1, np.concatenate([src, nodes, glob]), np.concatenate([co, glob, nodes]))


def papers_c5(seed: int = 17):
    """C5 (ogbn-papers100M shape): S = 1,048,576 at 14.55
    arcs/node -> E ~ 16M incl. loops; communities of 256, ids shuffled."""
    return community_graph(1048576, 14.55, community=256, intra=0.8, sigma=1.0, seed=seed)

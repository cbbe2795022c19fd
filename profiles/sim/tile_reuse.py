"""Reuse inside the tile kernels' tiles on the bench's C3 pattern: per tile
(community order, <= ROWS rows, <= 4096 edges), distinct neighbour columns and
the share of the tile's edges whose column is among its N most-referenced
columns (what a shared-memory stage of N K/V rows would serve)."""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2407_14106_b200.attention import community_order

info = {}
ro, co = bench.cached_workload("ecr", info)
ro = np.asarray(ro, np.int64); co = np.asarray(co, np.int64)
n = ro.shape[0] - 1
deg = np.diff(ro)
order, _ = community_order(ro, co)
blocks = info["_blocks"]
tile_pair = np.zeros(co.shape[0], bool)
for r0, c0 in blocks:
    for r in range(r0, r0 + 16):
        a = ro[r] + np.searchsorted(co[ro[r]:ro[r + 1]], c0)
        tile_pair[a:a + 16] = True
print("tile pairs", tile_pair.sum())
for ROWS in (32, 64, 128, 256):
    tiles, cur, e = [], [], 0
    for r in order:
        d = int(deg[r])
        if d > 1024: continue
        if len(cur) == ROWS or e + d > 4096 * ROWS // 128:
            tiles.append(cur); cur, e = [], 0
        cur.append(r); e += d
    if cur: tiles.append(cur)
    tot = 0; distinct = []; cov = {64: 0, 128: 0, 256: 0, 512: 0}; cov_nt = dict(cov); tot_nt = 0
    for t in tiles[::7]:
        idx = np.concatenate([np.arange(ro[r], ro[r + 1]) for r in t])
        cols = co[idx]; nt = ~tile_pair[idx]
        u, c = np.unique(cols, return_counts=True)
        distinct.append(len(u)); tot += len(cols); tot_nt += nt.sum()
        srt = np.sort(c)[::-1]
        for N in cov: cov[N] += srt[:N].sum()
        # non-tile edges: reuse among them
        u2, c2 = np.unique(cols[nt], return_counts=True)
        s2 = np.sort(c2)[::-1]
        for N in cov_nt: cov_nt[N] += s2[:N].sum()
    print(f"ROWS={ROWS}: tiles {len(tiles)} distinct cols/tile {np.mean(distinct):.0f} edges/tile {tot/len(tiles[::7]):.0f}",
          "cover all:", {N: round(v / tot, 3) for N, v in cov.items()},
          "cover non-tile:", {N: round(v / tot_nt, 3) for N, v in cov_nt.items()})

"""Simulate the slot utilisation of the tile kernels' schedule on the bench's
C3 pattern (run on the GPU box: the ECR layout is built on the device).

Model: per tile, 8 warps x 4 slots step in lockstep; a step gives every busy
slot EPL edges; a slot whose row ends refills from the tile's shared queue;
a warp runs while any of its slots is busy. Utilisation = edges / (warp
steps x 4 slots x EPL)."""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_2407_14106_b200.attention import community_order

info = {}
ro, co = bench.cached_workload("ecr", info)
ro = np.asarray(ro, np.int64); co = np.asarray(co, np.int64)
n = ro.shape[0] - 1
deg = np.diff(ro)
print("S", n, "E", co.shape[0], "deg mean %.2f max %d p99 %d" % (deg.mean(), deg.max(), np.percentile(deg, 99)))
order, ncomm = community_order(ro, co)
EPL, ROWS, CAP, HUB = 4, 128, 4096, 1024

def tiles_of(order, deg):
    tiles, cur, e = [], [], 0
    for r in order:
        d = int(deg[r])
        if d > HUB: continue
        pd = (d + 3) // 4 * 4
        if len(cur) == ROWS or e + pd > CAP:
            tiles.append(cur); cur, e = [], 0
        cur.append(r); e += pd
    if cur: tiles.append(cur)
    return [sorted(t, key=lambda r: -deg[r]) for t in tiles]

def simulate(tiles, deg, W=8, SL=4, epl=EPL):
    steps = 0
    for t in tiles:
        d = [int(deg[r]) for r in t]
        q = W * SL
        rem = [d[i] if i < len(d) else -1 for i in range(W * SL)]
        while True:
            active = False
            for w in range(W):
                sl = rem[w * SL:(w + 1) * SL]
                if all(x < 0 for x in sl): continue
                active = True; steps += 1
                for s in range(SL):
                    x = rem[w * SL + s]
                    if x < 0: continue
                    x -= epl
                    if x <= 0:
                        if q < len(d): x = d[q]; q += 1
                        else: x = -1
                    rem[w * SL + s] = x
            if not active: break
    return steps

tl = tiles_of(order, deg)
E = int(sum(deg[r] for t in tl for r in t))
st = simulate(tl, deg)
print("community order: tiles", len(tl), "edges", E, "warp-steps", st, "util %.3f" % (E / (st * 4 * EPL)))
tn = tiles_of(np.arange(n), deg)
st2 = simulate(tn, deg)
print("natural order: util %.3f" % (E / (st2 * 4 * EPL)))

"""Scheduling probe for the tracking pose backward: per (tile, quadrant) item, the number of list
entries some pixel of the 8x8 block takes (= the item's walk length), against the per-slot load of a
perfectly balanced grid (148 SMs x 24 resident single-warp CTAs).  Prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2403_16095_b200 import api  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 500000
ctx = api.Context(0)
K = bench.intrinsics()
m, poses = bench.build_scene(P)
ctx.upload(m)
start = bench.perturbed(poses[1], bench.OFFSET)
r = ctx.render(start, K)
W, H = K.width, K.height
tx_n, ty_n = (W + 15) // 16, (H + 15) // 16
tr, pp = ctx.render_tiles(tx_n * ty_n, r.num_pairs)
rs, prim, _, _ = ctx.render_record_full(W * H)
taken = np.zeros((tx_n * ty_n, 4), np.int64)
for t in range(tx_n * ty_n):
    a, b = tr[t]
    if b <= a:
        continue
    pos = {int(pid): i for i, pid in enumerate(pp[a:b])}
    x0, y0 = (t % tx_n) * 16, (t // tx_n) * 16
    for q in range(4):
        seen = set()
        for yy in range(y0 + 8 * (q >> 1), min(y0 + 8 * (q >> 1) + 8, H)):
            for xx in range(x0 + 8 * (q & 1), min(x0 + 8 * (q & 1) + 8, W)):
                pi = yy * W + xx
                seen.update(pos[int(p)] for p in prim[rs[pi]:rs[pi + 1]])
        taken[t, q] = len(seen)
items = taken.ravel()
slots = 148 * 24
out = {"primitives": P, "items": int(items.size), "taken_mean": float(items.mean()), "taken_max": int(items.max()),
       "taken_p99": float(np.percentile(items, 99)), "per_slot_load": float(items.sum() / slots),
       "longest_over_slot_load": float(items.max() / (items.sum() / slots)),
       "top10": sorted(items.tolist())[-10:], "list_len_max": int((tr[:, 1] - tr[:, 0]).max())}
print(json.dumps(out))

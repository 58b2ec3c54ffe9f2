"""Count (warp block, list entry) pairs that hold a contributor for several warp-block shapes on the
fp64 oracle's render record at configs[1] (used to choose the 8x8 two-pixel layout)."""
import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
import bench, oracle
from paper_2403_16095_b200 import api
m, poses = bench.build_scene(500000)
K = bench.intrinsics()
t=time.time()
r = oracle.render(m, bench.perturbed(poses[1], bench.OFFSET), K)
print('render', time.time()-t)
rs, prim, a, tr = r.record()
W, H = K.width, K.height
pix = np.repeat(np.arange(W*H), np.diff(rs.astype(np.int64)))
x = pix % W; y = pix // W
print('contributors', len(prim))
for bw, bh in ((8,4),(4,8),(8,8),(16,4),(16,8)):
    blk = (y // bh) * ((W + bw - 1)//bw) + x // bw
    key = prim.astype(np.int64) * 10**6 + blk
    nb = len(np.unique(key))
    print(bw, bh, 'block-pairs', nb, 'lane eff', len(prim)/(nb*bw*bh))

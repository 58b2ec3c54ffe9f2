"""Driver for ncu captures of the mapping path (bench.py's sliding_ba setup: 16 keyframes of a
~1M-Gaussian scene): `python tools/profile_map.py [iterations]`.  Not a bench line."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    from paper_2403_16095_b200 import abi, api
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    K = bench.intrinsics()
    m, poses = bench.build_scene(1000000, seed=0)
    ctx = api.Context(0)
    ctx.upload(m)
    kf = [3 * i for i in range(16)]
    for j, f in enumerate(kf):
        r = ctx.render(poses[f], K, None)
        c, d = bench.noisy(r.color, r.alpha_depth, f)
        ctx.frame_upload(j, c, d, K.width, K.height)
    mc = abi.defaults_mapper()
    mc.densify_interval = 0
    tc = abi.defaults_tracker()
    kposes = [bench.perturbed(poses[f], [0.001, 0, 0, 0.002, 0, 0]) if j else poses[f] for j, f in enumerate(kf)]
    trace, _ = ctx.sliding_ba(list(range(16)), kposes, kf, K, tc, mc, iters)
    print("sliding_ba", iters, trace, flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

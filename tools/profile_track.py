"""Small driver for ncu captures of the configs[1] tracking iteration (same scene, frames and start
poses as bench.py): `python tools/profile_track.py [iterations] [frames]`.  Not a bench line."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    from paper_2403_16095_b200 import abi, api
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    nframes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ctx = api.Context(0)
    K = bench.intrinsics()
    m, poses = bench.build_scene(500000)
    ctx.upload(m)
    for f in range(4):
        r = ctx.render(poses[f], K)
        c, d = bench.noisy(r.color, r.alpha_depth, f)
        ctx.frame_upload(f, c, d, K.width, K.height)
    ctx.accumulate_uncertainty([0, 1, 2, 3], poses[:4], K)
    ctx.prune_unreliable(0.025, 0.005)
    tc = abi.defaults_tracker()
    tc.iterations = iters
    for f in range(nframes):
        res = ctx.track_frame(1 + f % 3, bench.perturbed(poses[1 + f % 3], bench.OFFSET), K, tc, abi.defaults_weights(),
                              abi.defaults_raster())
        print(f, res.iterations_run, res.final_loss, flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

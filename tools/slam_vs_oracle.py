"""SlamSystem on the device vs the same pipeline over the fp64 oracle (oracle/slam.py, the
reference's SlamSystem::process control flow, system.cpp:31-154) on ONE reduced-resolution
sequence: is the trajectory drift / keyframe-PSNR fall of tools/bench_slam.py the reference's
behaviour at RunConfig defaults, or a device defect?

Frames: the reference room generator (~500k Gaussians) rendered on the device along the bench's
slow orbit (0.25 deg/frame) at 160x90 (Replica intrinsics scaled by 2/15) + NoiseSpec noise; both
arms consume the identical float32 frames.  Densification is off in both (its random draws are
exercised by tests/test_gpu_parity.py); everything else is RunConfig defaults (15 tracking
iterations per frame, a keyframe every 30 frames with 60 mapping iterations, sliding_ba 10,
uncertainty pruning, spawning).

Run on the GPU box:  python tools/slam_vs_oracle.py [frames] [port|reference] > gpurun_out/slam_vs_oracle.json
("reference": the oracle entry points route to the reference compiled from its unmodified sources,
oracle/_ref/libgsfref.so; the orchestration is oracle/slam.py's restatement of system.cpp either way)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from tools.bench_slam import ate_cm  # noqa: E402


def psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return 10.0 * np.log10(1.0 / max(mse, 1e-12))


def main():
    from paper_2403_16095_b200 import abi, api
    import oracle as orc
    from oracle.slam import OracleSlam
    from tools import synth
    nframes = int(sys.argv[1]) if len(sys.argv) > 1 else 91
    which = sys.argv[2] if len(sys.argv) > 2 else "port"
    s = 2.0 / 15.0
    K = api.intrinsics(600.0 * s, 600.0 * s, 599.5 * s, 339.5 * s, 160, 90, near_plane=0.1, far_plane=10.0)
    truth, _ = bench.build_scene(500000)
    poses = [api.pose_of(r, t) for r, t in synth.orbit(1440, 1.0, 0.0)]
    gen = api.Context(0)
    gen.upload(truth)
    frames = []
    for f in range(nframes):
        r = gen.render(poses[f], K)
        c, d = bench.noisy(r.color, r.alpha_depth, f)
        frames.append((np.ascontiguousarray(c, np.float32), np.ascontiguousarray(d, np.float32)))
    gen.close()

    def cfg():
        c = abi.defaults_slam(K)
        c.mapper.densify_interval = 0
        return c

    ctx = api.Context(0)
    slam = api.SlamSystem(ctx, cfg())
    t0 = time.perf_counter()
    dev = [slam.process(f, f / 30.0, c, d) for f, (c, d) in enumerate(frames)]
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    with orc.backend(which):
        ref = OracleSlam(cfg())
        ora = [ref.process(f, c, d) for f, (c, d) in enumerate(frames)]
    t_ora = time.perf_counter() - t0

    dev_poses = [l.pose for l in dev]
    kf_idx = [f for f, l in enumerate(dev) if l.keyframe]
    # keyframe PSNR of each arm's final map rendered at its own keyframe pose
    dev_psnr = [float(l.kf_psnr_db) for l in dev if l.keyframe]
    dev_final = [psnr(ctx.render(dev_poses[k], K).color, frames[k][0]) for k in kf_idx]
    ora_psnr = []
    with orc.backend(which):
        m = ref.st.get()
        for kf in ref.keyframes:
            rr = orc.render(m, kf["pose"], K)
            ora_psnr.append(psnr(rr.color, kf["rgb"]))
    per_frame = []
    for f in range(nframes):
        per_frame.append({
            "frame": f,
            "ate_dev_cm": ate_cm(dev_poses[: f + 1], poses[: f + 1]) if f else 0.0,
            "ate_oracle_cm": ate_cm(ora[: f + 1], poses[: f + 1]) if f else 0.0,
            "dev_vs_oracle_cm": float(np.linalg.norm(np.array(list(dev_poses[f].translation)) -
                                                     np.array(list(ora[f].translation))) * 100.0),
        })
    out = {
        "what": "SlamSystem device vs the fp64 oracle orchestration on the same frames (160x90, RunConfig defaults, "
                "densify off)", "oracle_backend": which,
        "frames": nframes, "keyframes": kf_idx,
        "ate_rmse_cm": {"device": ate_cm(dev_poses, poses[:nframes]), "oracle": ate_cm(ora, poses[:nframes])},
        "kf_psnr_db": {"device_at_keyframe_time": dev_psnr, "device_final_map": dev_final, "oracle_final_map": ora_psnr},
        "max_dev_vs_oracle_cm": max(p["dev_vs_oracle_cm"] for p in per_frame),
        "wall_s": {"device": t_dev, "oracle": t_ora},
        "per_frame": per_frame[::5],
    }
    print(json.dumps(out))
    slam.close()


if __name__ == "__main__":
    main()

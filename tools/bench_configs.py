"""Per-config measurements of SURVEY.md §8(d) beside the headline bench.py line (not bench lines):

  cfg1  100k Gaussians, 640x480 (f=525): one render + render_backward with mapping-loss seeds
        (all five maps, observed depth given) -> device ms per kernel class, algorithmic FP32
        fraction of the blend / backward; the CPU reference (oracle/_ref: the unmodified reference
        sources) on the same call sequence, median of 3
  cfg3  TUM-shaped 640x480 (fx 517.3), 200k, handheld_real weights: 30 frames, track_frame(25) each,
        map_step(45) over the last keyframes every 15 frames -> tracked frames/s, mapping it/s; the
        CPU reference's track_frame(1) - track_frame(0) and map_step(1) on the same scene beside it
  cfg4  sliding_ba over 16 keyframes of a ~1M-Gaussian scene: the CPU reference's sliding_ba(1)
        on 2 keyframes, scaled to the 16-keyframe window (the device number is bench.py's
        `mapping` object)
  cfg5  ScanNet-shaped 640x480 (fx 577.6), P in {10k .. 4M}: render + render_backward ms (device
        event brackets), the workload statistics V / M / T / C / longest tile list, and the
        algorithmic FP32 fraction of the blend / backward and HBM GB/s of the preprocess

  --ncu-sweep  one render + render_backward per cfg5 size and nothing else, separated by a tiny
               SSIM call, for `ncu --metrics ...` (tools/gpu/configs.sh); tools/ncu_sweep_parse.py
               attributes the launches to sizes and writes profiles/r02_cfg5_ncu.json

Run on the GPU box:  bash tools/gpu/configs.sh   (outputs under gpurun_out/, copied to profiles/)
Inputs are the reference room generator (synthetic.cpp:56-104, mt19937_64 seed 0, via tools/synth)
with the seeded anisotropy of SURVEY §8(d) and orbit poses; targets are device renders of the
ground truth plus the NoiseSpec noise (as bench.py).  The CPU legs render their own targets with the
reference from the same map (the device's fp32 map, downloaded)."""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (scene, noise and pose helpers shared with the headline bench)

SWEEP = (10000, 30000, 100000, 300000, 1000000, 2000000, 4000000)


def cam(fx, fy, cx, cy, w, h):
    from paper_2403_16095_b200.abi import Intrinsics
    return Intrinsics(fx, fy, cx, cy, w, h, 1.0, 0.1, 10.0)


def peaks():
    fp32, _ = bench.fp32_peak_measured()
    p, _ = bench.measured_peaks()
    return (fp32 or 73.9), float(p.get("hbm_gbs", 6451.8))


def profile(ctx, fn, reps=5):
    """Median device ms per kernel class over `reps` calls of fn (CUDA events on the library stream)."""
    classes = ("preprocess", "sort_binning", "blend", "backward", "chain")
    rows = []
    for _ in range(reps):
        ctx.lib.gsf_profile_enable(ctx.h, 1)
        ctx.lib.gsf_event_record(ctx.h, 0)
        fn()
        ctx.lib.gsf_event_record(ctx.h, 1)
        ms = C.c_double()
        ctx.lib.gsf_event_elapsed(ctx.h, 0, 1, C.byref(ms))
        row = {"wall_ms": ms.value}
        for k, name in enumerate(classes):
            t, n = C.c_double(), C.c_int64()
            ctx.lib.gsf_profile_read(ctx.h, k, C.byref(t), C.byref(n))
            row[name] = t.value
        ctx.lib.gsf_profile_enable(ctx.h, 0)
        rows.append(row)
    return {k: float(np.median([r[k] for r in rows])) for k in rows[0]}


def workload(ctx, r, K):
    """V, M, T (traversed (pixel, entry) pairs of the tile walk), C (contributors), longest list."""
    tx, ty = (K.width + 15) // 16, (K.height + 15) // 16
    tr, _ = ctx.render_tiles(tx * ty, r.num_pairs)
    ln = (tr[:, 1] - tr[:, 0]).astype(np.float64)
    pix = np.array([min(16, K.width - (t % tx) * 16) * min(16, K.height - (t // tx) * 16) for t in range(tx * ty)],
                   np.float64)
    return {"visible": int(r.num_visible), "pairs": int(r.num_pairs), "max_tile_list": int(ln.max()),
            "traversed_T": float((ln * pix).sum()), "contributors_C": float(r.per_pixel_count.sum())}


def fractions(wl, dev, P, fp32_peak, hbm_peak):
    """Algorithmic FP32 fractions of the blend (11 T + 24 C flops) and the backward (13 T + 70 C) —
    SURVEY §8(d)'s flop model — and the preprocess's algorithmic HBM GB/s (56 B of parameters read
    and one visibility byte per primitive; 120 B of records per visible primitive written)."""
    T, Cn = wl["traversed_T"], wl["contributors_C"]
    out = {}
    for k, fl in (("blend", 11.0 * T + 24.0 * Cn), ("backward", 13.0 * T + 70.0 * Cn)):
        ms = dev.get(k, 0.0)
        if ms > 0:
            tf = fl / (ms * 1e-3) / 1e12
            out[k] = {"algorithmic_gflop": fl / 1e9, "tflops": tf, "frac_fp32": tf / fp32_peak}
    ms = dev.get("preprocess", 0.0)
    if ms > 0:
        by = P * 57.0 + wl["visible"] * 120.0
        gbs = by / (ms * 1e-3) / 1e9
        out["preprocess"] = {"algorithmic_mb": by / 1e6, "gbs": gbs, "frac_hbm": gbs / hbm_peak}
    return out


def ref_kind():
    import oracle
    return "reference" if oracle.reference_available() else "port"


def cfg1(out):
    from paper_2403_16095_b200 import abi, api
    import oracle
    K = cam(525.0, 525.0, 319.5, 239.5, 640, 480)
    m, poses = bench.build_scene(100000)
    ctx = api.Context(0)
    ctx.upload(m)
    r = ctx.render(poses[3], K)
    tgt, obs = bench.noisy(r.color, r.alpha_depth, 3)
    p = bench.perturbed(poses[3], bench.OFFSET)
    w = abi.defaults_weights()

    def fwd_bwd():
        ctx.render(p, K, obs)
        _, (dc, dad, dmd, du, _) = ctx.evaluate_mapping_loss(tgt, obs, w)
        ctx.render_backward(dc.reshape(480, 640, 3), dad.reshape(480, 640), dmd.reshape(480, 640), None,
                            du.reshape(480, 640), obs)

    fwd_bwd()
    dev = profile(ctx, fwd_bwd)
    wl = workload(ctx, ctx.render(p, K, obs), K)
    mm = ctx.download()
    kind = ref_kind()
    cpu = []
    with oracle.backend(kind):
        ow = oracle.defaults_weights()
        for _ in range(3):
            t0 = time.perf_counter()
            o = oracle.render(mm, p, K, obs.astype(np.float64))
            loss, (dc, dad, dmd, du, dls) = oracle.mapping_loss(mm, o, tgt.astype(np.float64), obs.astype(np.float64),
                                                               K, ow)
            oracle.render_backward(mm, p, K, o, dc, dad, dmd, None, du, obs.astype(np.float64))
            cpu.append(time.perf_counter() - t0)
        threads = oracle.threads()
    fp32, hbm = peaks()
    kern_ms = dev["preprocess"] + dev["sort_binning"] + dev["blend"] + dev["backward"] + dev["chain"]
    out["cfg1"] = {"workload": "100k Gaussians, 640x480 f=525: render + mapping loss + render_backward (all maps)",
                   "primitives": int(m.count), "workload_stats": wl, "device_ms": dev,
                   "device_kernels_ms": kern_ms, "roofline": fractions(wl, dev, m.count, fp32, hbm),
                   "cpu_baseline": {"kind": kind, "s_median3": float(np.median(cpu)), "samples_s": cpu,
                                    "cores": threads, "sample": "render + evaluate_mapping_loss + render_backward, "
                                    "the same map / pose / target as the device call"},
                   "device_kernels_vs_cpu": float(np.median(cpu)) / (kern_ms * 1e-3)}
    ctx.close()


def cfg3(out):
    from paper_2403_16095_b200 import abi, api
    import oracle
    K = cam(517.3, 516.5, 318.6, 255.3, 640, 480)
    m, poses = bench.build_scene(200000)
    ctx = api.Context(0)
    ctx.upload(m)
    frames = []
    for f in range(30):
        r = ctx.render(poses[f], K)
        c, d = bench.noisy(r.color, r.alpha_depth, f)
        ctx.frame_upload(f, c, d, 640, 480)
        frames.append((c, d))
    tc = abi.defaults_tracker()
    tc.iterations = 25
    w = abi.defaults_weights(True)        # LossWeights::handheld_real (losses.cpp:35-46)
    mc = abi.defaults_mapper()
    mc.densify_interval = 0
    mc.weights = abi.defaults_weights(True)
    rc = abi.defaults_raster()
    mm = ctx.download()                   # the CPU leg's map (before mapping changes it)
    ctx.track_frame(0, poses[0], K, tc, w, rc)   # warm-up
    track_ms, track_dev_ms, map_ms, map_dev_ms, map_its = 0.0, 0.0, 0.0, 0.0, 0
    est = [poses[0]]
    ev = C.c_double()
    for f in range(1, 30):
        ctx.lib.gsf_synchronize(ctx.h)
        t0 = time.perf_counter()
        ctx.lib.gsf_event_record(ctx.h, 0)
        res = ctx.track_frame(f, bench.perturbed(est[-1], [0, 0, 0, 0, 0, 0]), K, tc, w, rc)
        ctx.lib.gsf_event_record(ctx.h, 1)
        track_ms += (time.perf_counter() - t0) * 1e3
        ctx.lib.gsf_event_elapsed(ctx.h, 0, 1, C.byref(ev))
        track_dev_ms += ev.value
        est.append(res.pose)
        if f % 15 == 0:
            win = list(range(max(0, f - 3), f + 1))
            ctx.lib.gsf_synchronize(ctx.h)
            t0 = time.perf_counter()
            ctx.lib.gsf_event_record(ctx.h, 2)
            ctx.map_step(win, [est[k] for k in win], K, mc, 45)
            ctx.lib.gsf_event_record(ctx.h, 3)
            map_ms += (time.perf_counter() - t0) * 1e3
            ctx.lib.gsf_event_elapsed(ctx.h, 2, 3, C.byref(ev))
            map_dev_ms += ev.value
            map_its += 45
    # CPU reference on the same scene: track_frame(1) - track_frame(0) per iteration, map_step(1)
    kind = ref_kind()
    c64, d64 = frames[1][0].astype(np.float64), frames[1][1].astype(np.float64)
    t1s, t0s, msteps = [], [], []
    with oracle.backend(kind):
        otc = oracle.defaults_tracker()
        ow = oracle.defaults_weights(True)
        orc = oracle.defaults_raster()
        start = bench.perturbed(poses[1], bench.OFFSET)
        for _ in range(3):
            otc.iterations = 1
            a = time.perf_counter()
            oracle.track_frame(mm, c64, d64, start, K, otc, ow, orc)
            t1s.append(time.perf_counter() - a)
            otc.iterations = 0
            a = time.perf_counter()
            oracle.track_frame(mm, c64, d64, start, K, otc, ow, orc)
            t0s.append(time.perf_counter() - a)
        omc = oracle.defaults_mapper()
        omc.densify_interval = 0
        omc.weights = oracle.defaults_weights(True)
        st = oracle.MapState(mm, omc)
        win = [(frames[k][0].astype(np.float64), frames[k][1].astype(np.float64)) for k in range(4)]
        for _ in range(2):
            a = time.perf_counter()
            st.map_step(win, poses[:4], K, omc, 1)
            msteps.append(time.perf_counter() - a)
        threads = oracle.threads()
    t_iter, t_final, hz = bench.extrapolate(t1s, t0s, 25)
    dev_hz = 29 / (track_dev_ms / 1e3)
    map_dev = map_its / (map_dev_ms / 1e3)
    out["cfg3"] = {"workload": "TUM-shaped 640x480, 200k, handheld_real weights: 29 tracked frames x 25 iterations, "
                               "map_step(45) every 15 frames (4-keyframe window)",
                   "primitives": int(m.count), "tracking_frames_per_s": dev_hz,
                   "tracking_ms_per_iter": track_dev_ms / (29 * 25),
                   "tracking_frames_per_s_wall": 29 / (track_ms / 1e3), "mapping_it_per_s": map_dev,
                   "mapping_it_per_s_wall": map_its / (map_ms / 1e3),
                   "timing": "CUDA events on the library stream around each track_frame / map_step call (wall clock "
                             "beside it)",
                   "cpu_baseline": {"kind": kind, "cores": threads, "tracking_frames_per_s": hz,
                                    "tracking_s_per_iter": t_iter, "mapping_it_per_s": 1.0 / float(np.median(msteps)),
                                    "sample": "3 x track_frame(1) / track_frame(0) on frame 1 (25 iterations "
                                              "extrapolated), 2 x map_step(1) over a 4-keyframe window",
                                    "samples_s": {"track1": t1s, "track0": t0s, "map_step1": msteps}},
                   "vs_cpu": {"tracking": dev_hz / hz, "mapping": map_dev * float(np.median(msteps))}}
    ctx.close()


def cfg4_cpu(out):
    """The CPU reference's sliding_ba iteration over a 2-keyframe slice of the cfg4 window, scaled to
    16 keyframes (per keyframe the reference renders, evaluates and back-propagates once; the Adam
    step over the map is counted once)."""
    from paper_2403_16095_b200 import api
    import oracle
    K = bench.intrinsics()
    m, poses = bench.build_scene(1000000)
    ctx = api.Context(0)
    ctx.upload(m)
    kf = [0, 3]
    frames = []
    for f in kf:
        r = ctx.render(poses[f], K)
        c, d = bench.noisy(r.color, r.alpha_depth, f)
        frames.append((c.astype(np.float64), d.astype(np.float64)))
    mm = ctx.download()
    ctx.close()
    kind = ref_kind()
    with oracle.backend(kind):
        omc = oracle.defaults_mapper()
        omc.densify_interval = 0
        otc = oracle.defaults_tracker()
        st = oracle.MapState(mm, omc)
        kp = [poses[0], bench.perturbed(poses[3], [0.001, 0, 0, 0.002, 0, 0])]
        ts = []
        for n in (1, 2):
            a = time.perf_counter()
            st.sliding_ba(frames[:n], kp[:n], kf[:n], K, otc, omc, 1)
            ts.append(time.perf_counter() - a)
        threads = oracle.threads()
    per_kf = max(ts[1] - ts[0], 1e-9)
    fixed = max(ts[0] - per_kf, 0.0)
    it_s = fixed + 16 * per_kf
    out["cfg4_cpu"] = {"workload": "sliding_ba iteration, 16-keyframe window, ~1M Gaussians, 1200x680",
                       "primitives": int(m.count), "kind": kind, "cores": threads,
                       "sample": "sliding_ba(1) over 1 and 2 keyframes; per keyframe = the difference, the "
                                 "16-keyframe iteration = the 1-keyframe fixed part + 16 x that",
                       "samples_s": ts, "s_per_iter_16kf": it_s, "it_per_s": 1.0 / it_s}


def cfg5(out):
    from paper_2403_16095_b200 import api
    K = cam(577.6, 578.7, 318.9, 242.7, 640, 480)
    rows = []
    rng = np.random.default_rng(5)
    fp32, hbm = peaks()
    for P in SWEEP:
        m, poses = bench.build_scene(P)
        ctx = api.Context(0)
        ctx.upload(m)
        p = poses[5]
        up = [rng.standard_normal((480, 640, 3)).astype(np.float32), rng.standard_normal((480, 640)).astype(np.float32)]

        def fwd_bwd():
            ctx.render(p, K)
            ctx.render_backward(up[0], up[1])

        fwd_bwd()
        wl = workload(ctx, ctx.render(p, K), K)
        dev = profile(ctx, fwd_bwd)
        rows.append({"primitives": int(m.count), **wl, "device_ms": dev,
                     "roofline": fractions(wl, dev, m.count, fp32, hbm)})
        ctx.close()
    out["cfg5"] = {"workload": "ScanNet-shaped 640x480 sweep: render + render_backward (explicit upstream colour "
                               "and alpha-depth maps)", "peaks": {"fp32_tflops": fp32, "hbm_gbs": hbm}, "rows": rows}


def ncu_sweep():
    """Launch sequence for ncu: per size one render + render_backward after a warm-up call, sizes
    separated by a 16x16 SSIM call (k_ssim_* launches mark the boundaries)."""
    from paper_2403_16095_b200 import api
    K = cam(577.6, 578.7, 318.9, 242.7, 640, 480)
    rng = np.random.default_rng(5)
    x = rng.random((16, 16, 3)).astype(np.float32)
    for P in SWEEP:
        m, poses = bench.build_scene(P)
        ctx = api.Context(0)
        ctx.upload(m)
        up = [rng.standard_normal((480, 640, 3)).astype(np.float32), rng.standard_normal((480, 640)).astype(np.float32)]
        ctx.render(poses[5], K)
        ctx.render_backward(up[0], up[1])
        ctx.ssim(x, x, 16, 16)      # boundary marker: the measured call follows
        ctx.render(poses[5], K)
        ctx.render_backward(up[0], up[1])
        ctx.ssim(x, x, 16, 16)
        ctx.close()
        print(json.dumps({"size": P, "primitives": int(m.count)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg3,cfg4_cpu,cfg5")
    ap.add_argument("--ncu-sweep", action="store_true")
    a = ap.parse_args()
    if a.ncu_sweep:
        ncu_sweep()
        return
    out = {"note": "SURVEY.md §8(d) per-config measurements; device_ms = CUDA-event brackets per kernel class "
                   "(median of 5 calls, wall_ms includes the API's host transfers)"}
    fns = {"cfg1": cfg1, "cfg3": cfg3, "cfg4_cpu": cfg4_cpu, "cfg5": cfg5}
    for name in a.only.split(","):
        t0 = time.perf_counter()
        fns[name](out)
        out.setdefault("elapsed_s", {})[name] = time.perf_counter() - t0
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

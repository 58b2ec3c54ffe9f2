"""Device runs of the runtime configuration branches and of the reference's loop-behaviour tests.

* RasterConfig is a runtime value (raster/config.hpp:5-16): the alpha clamp and its gradient stop
  (rasterizer.cpp:114, :451) on saturated scenes (opacities up to 0.999), gradcheck's smooth
  config (gradcheck.cpp:21-27: no skip, no termination, footprint sigma 8), a non-default clamp /
  dilation / termination / footprint, and uncertainty_full_gradient = false (rasterizer.cpp:362-363)
  — forward bit-exact vs the fp32 mirror and within the fp64 bars, backward vs fp64.
* Inputs that are NOT fp32-representable (the drop-in converts the caller's doubles to fp32): the
  integer-output mismatch rate against fp64 on the raw doubles is reported and bounded.
* Loop behaviour (test_tracker.cpp:286-317, :365-409; test_map.cpp:134-155, :213-244) on the
  device: gauge equivariance of tracking, BA pulling drifted poses back with a frozen anchor
  (trace compared with the fp64 oracle's), the 2-view nu = 0.115 window, a multi-view
  multi-primitive window against fp64, and a floating outlier flagged and pruned.
"""
import math

import numpy as np
import pytest

from helpers import (f32_round, logit, make_intrinsics, one_pixel_camera, perturbed, pose, rotation_error, scene,
                     to_api_map, translation_error)

pytestmark = pytest.mark.gpu


def _cfgs(orc):
    from paper_2403_16095_b200.abi import defaults_raster
    out = []
    c = defaults_raster()
    out.append(("default", c))
    c = defaults_raster()
    c.alpha_skip, c.termination_threshold, c.footprint_sigma = 0.0, 0.0, 8.0
    out.append(("smooth (gradcheck.cpp:21-27)", c))
    c = defaults_raster()
    c.alpha_clamp, c.dilation = 0.9, 0.1
    out.append(("clamp 0.9, dilation 0.1", c))
    c = defaults_raster()
    c.termination_threshold, c.footprint_sigma, c.alpha_skip = 1e-4, 2.5, 0.01
    out.append(("termination 1e-4, sigma 2.5, skip 0.01", c))
    c = defaults_raster()
    c.uncertainty_full_gradient = 0
    out.append(("uncertainty_full_gradient false", c))
    return out


def _saturated(orc, seed, P=300):
    m = orc.random_scene(seed, P, 1 if seed % 2 else 4, 0.999, 0.05, 0.25)
    rng = np.random.default_rng(seed)
    hi = rng.random(P) < 0.5
    m.opacity_logit[hi] = np.log(0.999 / 0.001) - rng.random(hi.sum()) * 1.5   # sigma in (0.995, 0.999)
    return f32_round(m)


def test_runtime_configs_forward(gpu_ctx, orc):
    rng = np.random.default_rng(8)
    for name, cfg in _cfgs(orc):
        for seed in range(3):
            m = _saturated(orc, 40 + seed)
            K = make_intrinsics(64, 48, 55.0)
            obs = orc.wavy_depth(64, 48, 2.5).astype(np.float32)
            p = pose(0.02 * rng.standard_normal(3), 0.03 * rng.standard_normal(3))
            gpu_ctx.upload(to_api_map(m))
            r = gpu_ctx.render(p, K, obs, cfg)
            mr = orc.mirror_render(m, p, K, obs, cfg)
            tr, pp = gpu_ctx.render_tiles(12, r.num_pairs)
            assert (tr.ravel() == mr.tile_range).all() and (pp == mr.rank_to_id[mr.pair_rank]).all(), name
            for k in ("per_pixel_count", "dominant", "median_prim", "median_valid"):
                assert (getattr(r, k) == getattr(mr, k)).all(), (name, k)
            for k in ("color", "alpha_depth", "median_depth", "opacity", "uncertainty", "final_transmittance"):
                assert np.array_equal(getattr(r, k), getattr(mr, k)), (name, k)
            o = orc.render(m, p, K, obs.astype(np.float64), cfg)
            for k in ("per_pixel_count", "dominant", "median_prim", "median_valid"):
                assert (getattr(r, k) == getattr(o, k)).all(), (name, k)
            for k in ("color", "alpha_depth", "opacity", "uncertainty", "final_transmittance"):
                assert np.abs(getattr(r, k) - getattr(o, k)).max() < 1e-4, (name, k)
            if name == "default" and seed == 0:
                _, prim, alpha, _ = o.record()
                assert (alpha == cfg.alpha_clamp).sum() > 50   # the clamp branch is exercised


def _grad_close(g, ref, rel, median, name):
    g = np.asarray(g, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    if np.abs(ref).max() == 0:
        assert np.abs(g).max() == 0, name
        return 0.0
    scale = np.maximum(np.abs(ref), 1e-3 * np.abs(ref).max())
    err = np.abs(g - ref) / scale
    assert err.max() <= rel, f"{name}: worst {err.max():.3e} at {err.argmax()}"
    assert np.median(err[ref != 0]) <= median, f"{name}: median {np.median(err[ref != 0]):.3e}"
    return float(err.max())


def test_runtime_configs_backward(gpu_ctx, orc):
    rng = np.random.default_rng(9)
    worst = {}
    for name, cfg in _cfgs(orc):
        for seed in range(3):
            m = _saturated(orc, 60 + seed, 150)
            K = make_intrinsics(48, 40, 45.0)
            obs = orc.wavy_depth(48, 40, 2.5).astype(np.float32)
            p = pose(0.02 * rng.standard_normal(3), 0.03 * rng.standard_normal(3))
            probe = [a.astype(np.float32).astype(np.float64) for a in
                     (rng.standard_normal((40, 48, 3)), rng.standard_normal((40, 48)), rng.standard_normal((40, 48)),
                      rng.standard_normal((40, 48)), rng.standard_normal((40, 48)))]
            gpu_ctx.upload(to_api_map(m))
            gpu_ctx.render(p, K, obs, cfg)
            g = gpu_ctx.render_backward(probe[0], probe[1], probe[2], probe[3], probe[4], obs)
            o = orc.render(m, p, K, obs.astype(np.float64), cfg)
            go = orc.render_backward(m, p, K, o, probe[0], probe[1], probe[2], probe[3], probe[4],
                                     obs.astype(np.float64), cfg)
            for k in ("d_mean", "d_log_scale", "d_quat", "d_opacity_logit", "d_sh", "d_mean2d"):
                e = _grad_close(getattr(g, k), getattr(go, k), 1e-3, 1e-5, f"{name} {k} seed {seed}")
                worst[name] = max(worst.get(name, 0.0), e)
            assert np.abs(g.d_pose - go.d_pose).max() <= 1e-4 * np.abs(go.d_pose).max(), name
    print("\nworst gradient rel err per config:", worst)


def test_uncertainty_full_gradient_false_drops_the_u_seed(gpu_ctx, orc):
    """rasterizer.cpp:362-363: with the flag off the uncertainty map is a stop-gradient statistic, so a
    seed on it alone yields an all-zero bundle (and no observed depth is needed)."""
    from paper_2403_16095_b200.abi import defaults_raster
    m = _saturated(orc, 77, 100)
    K = make_intrinsics(40, 30, 35.0)
    obs = orc.wavy_depth(40, 30, 2.5).astype(np.float32)
    cfg = defaults_raster()
    cfg.uncertainty_full_gradient = 0
    gpu_ctx.upload(to_api_map(m))
    gpu_ctx.render(pose(), K, obs, cfg)
    g = gpu_ctx.render_backward(d_uncertainty=np.ones((30, 40)), observed_depth=obs)
    assert (g.d_mean == 0).all() and (g.d_opacity_logit == 0).all() and (g.d_pose == 0).all()
    cfg.uncertainty_full_gradient = 1
    gpu_ctx.render(pose(), K, obs, cfg)
    g = gpu_ctx.render_backward(d_uncertainty=np.ones((30, 40)), observed_depth=obs)
    assert np.abs(g.d_mean).max() > 0


def test_raw_double_inputs_integer_mismatch_rate(gpu_ctx, orc):
    """The device stores the map in fp32; a caller's arbitrary doubles are rounded once at upload.
    Against fp64 on the RAW doubles the discrete outputs can then flip where a decision sits within
    fp32 rounding of a threshold (rho = 9 cutoff, alpha = 1/255 skip, depth ties).  Measured here on
    a 640x480 frame of 6,000 raw-double primitives: the rate is reported and must stay below 1e-4 of
    pixels; with fp32-representable inputs it is exactly zero (test_forward_vs_fp64_oracle)."""
    m = orc.random_scene(4242, 6000, 1, 0.95, 0.01, 0.08)
    K = make_intrinsics(640, 480, 525.0)
    gpu_ctx.upload(to_api_map(m))
    r = gpu_ctx.render(pose(), K)
    o = orc.render(m, pose(), K)
    mism = {k: int((getattr(r, k) != getattr(o, k)).sum()) for k in ("per_pixel_count", "dominant", "median_prim")}
    vis = int((r.visible != o.visible).sum())
    print(f"\nraw doubles: integer mismatches {mism} over {640 * 480} pixels, visible flags {vis} of 6000; "
          f"max colour err {np.abs(r.color - o.color).max():.2e}")
    assert all(v <= 1e-4 * 640 * 480 for v in mism.values()), mism
    assert np.abs(r.color - o.color).max() < 1e-3


# ---- loop behaviour -----------------------------------------------------------------------------
def _quat_mul(a, b):
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def _compose(a, b):
    """CameraPose::compose (pose.hpp:28-32): a after b."""
    from scipy.spatial.transform import Rotation as R
    ra, rb = R.from_rotvec(list(a.rotation_tangent)), R.from_rotvec(list(b.rotation_tangent))
    t = ra.apply(np.array(list(b.translation))) + np.array(list(a.translation))
    return pose((ra * rb).as_rotvec(), t)


def _inverse(a):
    from scipy.spatial.transform import Rotation as R
    ra = R.from_rotvec(list(a.rotation_tangent))
    return pose(-np.array(list(a.rotation_tangent)), -ra.inv().apply(np.array(list(a.translation))))


def test_tracking_gauge_equivariance(gpu_ctx, orc):
    """test_tracker.cpp:286-317 on the device: tracking in a rigidly re-expressed world returns the
    same camera.  The moved map is re-rounded to fp32, so the bar is fp32-scale (1e-4)."""
    from scipy.spatial.transform import Rotation as R
    from paper_2403_16095_b200.abi import defaults_tracker, defaults_weights
    prims = f32_round(orc.random_scene(23, 40))
    K = make_intrinsics(40, 30, 35.0)
    gpu_ctx.upload(to_api_map(prims))
    ob = gpu_ctx.render(pose(), K)
    gpu_ctx.frame_upload(0, ob.color, ob.alpha_depth, 40, 30)
    start = perturbed(pose(), [0.003, -0.002, 0.001, 0.006, 0.004, -0.005])
    tc = defaults_tracker()
    tc.iterations = 10
    w = defaults_weights(True)
    plain = gpu_ctx.track_frame(0, start, K, tc, w)
    gauge = pose((0.3, -0.2, 0.5), (0.4, -0.1, 0.25))
    rg = R.from_rotvec([0.3, -0.2, 0.5])
    th = np.linalg.norm([0.3, -0.2, 0.5])
    qg = np.r_[math.cos(0.5 * th), math.sin(0.5 * th) * np.array([0.3, -0.2, 0.5]) / th]
    moved = f32_round(prims)
    moved.mean = rg.apply(prims.mean) + np.array([0.4, -0.1, 0.25])
    moved.quat = np.array([_quat_mul(qg, q) for q in prims.quat])
    moved = f32_round(moved)
    gpu_ctx.upload(to_api_map(moved))
    gauged = gpu_ctx.track_frame(0, _compose(start, _inverse(gauge)), K, tc, w)
    back = _compose(gauged.pose, gauge)
    print(f"\ngauge: {rotation_error(back, plain.pose):.2e} rad, {translation_error(back, plain.pose):.2e} m")
    assert rotation_error(back, plain.pose) < 1e-4 and translation_error(back, plain.pose) < 1e-4


def test_ba_pulls_drifted_poses_back_with_frozen_anchor(gpu_ctx, orc):
    """test_tracker.cpp:365-409 on the device, on the reference test's own scene (textured_wall(20, 15)
    from std::mt19937(41), helpers.textured_wall) and frames (the fp64 render at the true poses): 25
    sliding_ba iterations with the full mapping objective must cut the window pose error below 0.4x
    and leave the anchor untouched; the device's loss trace is reported next to the fp64 oracle's."""
    from paper_2403_16095_b200.abi import defaults_mapper, defaults_tracker
    from helpers import textured_wall
    wall = textured_wall(20, 15, 41)
    K = make_intrinsics(48, 36, 40.0)
    truth = [pose(), perturbed(pose(), [0.02, -0.01, 0.0, 0.06, 0.02, -0.03]),
             perturbed(pose(), [-0.01, 0.02, 0.01, -0.05, 0.04, 0.03])]
    frames = []
    for i, t in enumerate(truth):
        ob = orc.render(wall, t, K)
        frames.append((ob.color.copy(), ob.alpha_depth.copy()))
        gpu_ctx.frame_upload(i, ob.color, ob.alpha_depth, 48, 36)
    kp = [truth[0], perturbed(truth[1], [0.006, -0.004, 0.003, 0.008, -0.006, 0.005]),
          perturbed(truth[2], [-0.005, 0.003, -0.004, -0.007, 0.008, -0.006])]
    err_before = sum(rotation_error(kp[i], truth[i]) + translation_error(kp[i], truth[i]) for i in (1, 2))
    mc = defaults_mapper()
    mc.densify_interval = 0
    tc = defaults_tracker()
    gpu_ctx.upload(to_api_map(wall))
    trace, out = gpu_ctx.sliding_ba([0, 1, 2], kp, [0, 10, 20], K, tc, mc, 25)
    err_after = sum(rotation_error(out[i], truth[i]) + translation_error(out[i], truth[i]) for i in (1, 2))
    st = orc.MapState(wall, mc)
    otrace, oout = st.sliding_ba(frames, kp, [0, 10, 20], K, tc, mc, 25)
    oerr = sum(rotation_error(oout[i], truth[i]) + translation_error(oout[i], truth[i]) for i in (1, 2))
    print(f"\nBA drift (reference scene): window pose error {err_before:.4e} -> device {err_after:.4e} "
          f"({err_after / err_before:.3f}x), fp64 {oerr:.4e} ({oerr / err_before:.3f}x); trace device "
          f"{np.round(trace[[0, 4, 9, 14, 19, 24]], 5)}, fp64 {np.round(otrace[[0, 4, 9, 14, 19, 24]], 5)}")
    assert err_after < 0.4 * err_before and trace[-1] < trace[0]
    assert list(out[0].rotation_tangent) == list(kp[0].rotation_tangent)
    assert list(out[0].translation) == list(kp[0].translation)
    assert trace[0] == pytest.approx(otrace[0], rel=1e-5)


def _dominant_weight_pose(orc, m, K, target_w):
    """A pure camera-x translation that puts the primitive's dominant weight at target_w (fp64 bisection)."""
    lo, hi = 0.0, 1.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        w = orc.render(m, pose((0, 0, 0), (mid, 0, 0)), K).dominant_weight[0, 0]
        lo, hi = (mid, hi) if w > target_w else (lo, mid)
    return pose((0, 0, 0), (0.5 * (lo + hi), 0, 0))


def test_uncertainty_two_view_window(gpu_ctx, orc):
    """test_map.cpp:134-155 on the device: views with dominant weights 0.9 and 0.5 and residuals 0.5 /
    0.1 give nu = (0.225 + 0.005) / 2 = 0.115 in either window order."""
    K = one_pixel_camera()
    m = f32_round(scene([dict(mean=[0, 0, 1.5], scale=0.1, opacity=0.9, color=[0.5, 0.5, 0.5])]))
    pb = _dominant_weight_pose(orc, m, K, 0.5)
    gpu_ctx.upload(to_api_map(m))
    gpu_ctx.frame_upload(0, np.zeros(3), np.array([2.0]), 1, 1)
    gpu_ctx.frame_upload(1, np.zeros(3), np.array([1.6]), 1, 1)
    assert gpu_ctx.accumulate_uncertainty([0, 1], [pose(), pb], K) == 1
    nu_ab = gpu_ctx.download().uncertainty[0]
    gpu_ctx.upload(to_api_map(m))
    gpu_ctx.accumulate_uncertainty([1, 0], [pb, pose()], K)
    nu_ba = gpu_ctx.download().uncertainty[0]
    assert nu_ab == pytest.approx(0.115, abs=2e-7) and nu_ba == pytest.approx(nu_ab, rel=1e-14)


def test_uncertainty_window_vs_fp64(gpu_ctx, orc):
    """accumulate_uncertainty + prune_unreliable (uncertainty.cpp:17-100) over a 4-view window of a
    300-primitive scene: nu within 1e-5 relative of fp64, observed flags and prune decisions equal."""
    m = f32_round(orc.random_scene(515, 300, 1, 0.99))
    K = make_intrinsics(64, 48, 55.0)
    poses = [pose(), pose((0.0, 0.03, 0.0), (0.02, 0.0, 0.0)), pose((0.02, 0.0, 0.0), (0.0, -0.02, 0.0)),
             pose((-0.01, -0.02, 0.01), (0.01, 0.01, 0.03))]
    depths = [orc.wavy_depth(64, 48, 2.2 + 0.2 * i).astype(np.float32) for i in range(4)]
    gpu_ctx.upload(to_api_map(m))
    for i, d in enumerate(depths):
        gpu_ctx.frame_upload(i, np.zeros((48, 64, 3)), d, 64, 48)
    n = gpu_ctx.accumulate_uncertainty([0, 1, 2, 3], poses, K)
    red = gpu_ctx.prune_unreliable(0.025, 0.005)
    g = gpu_ctx.download()
    om = f32_round(m)
    rs = [orc.render(om, p, K, d.astype(np.float64)) for p, d in zip(poses, depths)]
    on = orc.accumulate_uncertainty(om, rs, [d.astype(np.float64) for d in depths], poses, K)
    ored = orc.prune_unreliable(om, 0.025, 0.005)
    print(f"\nuncertainty window: observed {n} vs {on}, pruned {red} vs {ored}, max nu rel err "
          f"{np.max(np.abs(g.uncertainty - om.uncertainty) / np.maximum(om.uncertainty, 1e-12)):.2e}")
    assert n == on and red == ored
    assert (g.observed == om.observed).all()
    assert np.allclose(g.uncertainty, om.uncertainty, rtol=1e-5, atol=1e-12)
    assert np.array_equal(g.opacity_logit < -5, om.opacity_logit < -5)


def test_floating_outlier_flagged_and_pruned(gpu_ctx, orc):
    """test_map.cpp:213-244 on the device: a primitive pulled off a wall toward the camera gets
    nu > tau within one cycle and is pruned to opacity 0.005; the wall survives."""
    prims = [dict(mean=[0.25 * gx, 0.25 * gy, 2.0], scale=0.14, opacity=0.9, color=[0.5, 0.5, 0.5])
             for gy in range(-3, 4) for gx in range(-3, 4)]
    prims.append(dict(mean=[0.1, 0.05, 1.5], scale=0.14, opacity=0.9, color=[0.5, 0.5, 0.5]))
    m = f32_round(scene(prims))
    K = make_intrinsics(48, 36, 40.0)
    gpu_ctx.upload(to_api_map(m))
    gpu_ctx.frame_upload(0, np.zeros((36, 48, 3)), np.full((36, 48), 2.0), 48, 36)
    gpu_ctx.accumulate_uncertainty([0], [pose()], K)
    d = gpu_ctx.download()
    outlier = len(prims) - 1
    assert d.observed[outlier] == 1 and d.uncertainty[outlier] > 0.025
    assert gpu_ctx.prune_unreliable(0.025, 0.005) >= 1
    d = gpu_ctx.download()
    op = 1 / (1 + np.exp(-d.opacity_logit))
    assert op[outlier] == pytest.approx(0.005, rel=1e-5)
    assert (op[:outlier] >= 0.01).all()


def test_ba_first_step_matches_fp64(gpu_ctx, orc):
    """sliding_ba's first iteration on the textured-wall window: the per-keyframe mapping-loss pose
    gradients (render -> evaluate_mapping_loss -> render_backward, tracker.cpp:148-166) against fp64,
    and the first Adam step of every window pose and parameter (+-lr times the gradient's sign)."""
    from paper_2403_16095_b200.abi import defaults_mapper, defaults_tracker, defaults_weights
    from helpers import textured_wall
    prims = f32_round(textured_wall(20, 15, 41))
    K = make_intrinsics(48, 36, 40.0)
    truth = [pose(), perturbed(pose(), [0.02, -0.01, 0.0, 0.06, 0.02, -0.03]),
             perturbed(pose(), [-0.01, 0.02, 0.01, -0.05, 0.04, 0.03])]
    gpu_ctx.upload(to_api_map(prims))
    frames = []
    for i, t in enumerate(truth):
        ob = gpu_ctx.render(t, K)
        frames.append((ob.color.copy(), ob.alpha_depth.copy()))
        gpu_ctx.frame_upload(i, ob.color, ob.alpha_depth, 48, 36)
    kp = [truth[0], perturbed(truth[1], [0.006, -0.004, 0.003, 0.008, -0.006, 0.005]),
          perturbed(truth[2], [-0.005, 0.003, -0.004, -0.007, 0.008, -0.006])]
    w = defaults_weights()
    worst = 0.0
    for i in (1, 2):
        c, d = frames[i]
        gpu_ctx.render(kp[i], K, d)
        lm, (dc, dad, dmd, du, dls) = gpu_ctx.evaluate_mapping_loss(c, d, w)
        g = gpu_ctx.render_backward(dc.reshape(36, 48, 3), dad.reshape(36, 48), dmd.reshape(36, 48), None,
                                    du.reshape(36, 48), d)
        o = orc.render(prims, kp[i], K, d.astype(np.float64))
        om, (odc, odad, odmd, odu, odls) = orc.mapping_loss(prims, o, c.astype(np.float64), d.astype(np.float64), K, w)
        go = orc.render_backward(prims, kp[i], K, o, d_color=odc.reshape(36, 48, 3), d_alpha_depth=odad.reshape(36, 48),
                                 d_median_depth=odmd.reshape(36, 48), d_uncertainty=odu.reshape(36, 48),
                                 obs=d.astype(np.float64))
        rel = float(np.abs(g.d_pose - go.d_pose).max() / np.abs(go.d_pose).max())
        worst = max(worst, rel)
        print(f"\nkeyframe {i}: loss {lm.total:.9g} vs {om.total:.9g}; d_pose {g.d_pose} vs {go.d_pose} ({rel:.2e})")
        assert lm.total == pytest.approx(om.total, rel=1e-5)
    assert worst < 1e-3
    mc = defaults_mapper()
    mc.densify_interval = 0
    tc = defaults_tracker()
    gpu_ctx.upload(to_api_map(prims))
    trace, out = gpu_ctx.sliding_ba([0, 1, 2], kp, [0, 10, 20], K, tc, mc, 1)
    st = orc.MapState(prims, mc)
    otrace, oout = st.sliding_ba([(c.astype(np.float64), d.astype(np.float64)) for c, d in frames], kp, [0, 10, 20], K,
                                 tc, mc, 1)
    for a, b in zip(out, oout):
        assert np.abs(np.r_[list(a.rotation_tangent), list(a.translation)] -
                      np.r_[list(b.rotation_tangent), list(b.translation)]).max() < 1e-9
    assert trace[0] == pytest.approx(otrace[0], rel=1e-5)


def _list_extent(ctx, p, K):
    r = ctx.render(p, K)
    ntiles = ((K.width + 15) // 16) * ((K.height + 15) // 16)
    tr, _ = ctx.render_tiles(ntiles, r.num_pairs)
    return int((tr[:, 1] - tr[:, 0]).max()), int(r.num_pairs)


def _cluster_scene(orc):
    """random_scene(901, 400) plus 200 small primitives at (-0.52, 0.1, 1.5): outside the 64x48
    f=90 view from a camera 8 cm to the -x side, inside it from the identity pose.  Tracking from
    that start toward the identity brings the cluster into view mid-loop (fp64 oracle: lists
    (89 longest, 938 pairs) at the start, (274, 1245) after 40 iterations, (272, 1235) after 60)."""
    from types import SimpleNamespace
    base = orc.random_scene(901, 400)
    rng = np.random.default_rng(5)
    cl = scene([dict(mean=[-0.52 + 0.004 * rng.standard_normal(), 0.1 + 0.004 * rng.standard_normal(), 1.5],
                     scale=0.006, opacity=0.3, color=[0.9, 0.2, 0.1]) for _ in range(200)])
    return f32_round(SimpleNamespace(**{k: np.concatenate([getattr(base, k), getattr(cl, k)])
                                        for k in ("mean", "log_scale", "quat", "opacity_logit", "sh", "uncertainty",
                                                  "observed")}))


def test_overflow_mid_loop_grows_and_matches(gpu_ctx, orc):
    """A tracking loop whose lists peak mid-loop (a cluster enters the view as the camera moves),
    with the binning capacities reserved to fit the START render exactly: the captured loop
    overflows only after it began.  track_frame must retry with the loop's maxima (DevState M_max /
    max_tile), grow, and return the same pose bit for bit as a run that never overflowed — never a
    pose from truncated lists.  The API render and tracking_gradient paths grow the same way."""
    from paper_2403_16095_b200.abi import defaults_raster, defaults_tracker, defaults_weights
    K = make_intrinsics(64, 48, 90.0)
    m = _cluster_scene(orc)
    gpu_ctx.upload(to_api_map(m))
    gt = gpu_ctx.render(pose(), K)
    gpu_ctx.frame_upload(0, gt.color, gt.alpha_depth, 64, 48)
    tc = defaults_tracker()
    tc.iterations = 60
    w = defaults_weights(True)
    start = perturbed(pose(), [0, 0, 0, -0.08, 0, 0])
    ref = gpu_ctx.track_frame(0, start, K, tc, w)                 # default capacities: no overflow
    L0, M0 = _list_extent(gpu_ctx, start, K)
    L1, M1 = _list_extent(gpu_ctx, ref.pose, K)
    assert L1 > L0 + 100 and M1 > M0 + 100, (L0, M0, L1, M1)     # the cluster entered mid-loop
    ores = orc.track_frame(m, gt.color.astype(np.float64), gt.alpha_depth.astype(np.float64), start, K, tc, w,
                           defaults_raster())
    assert translation_error(ref.pose, ores.pose) < 2e-3 and rotation_error(ref.pose, ores.pose) < 2e-3
    gpu_ctx.reserve(M0, L0)
    assert gpu_ctx.capacity() == (max(M0, 64), max(L0, 32))
    assert _list_extent(gpu_ctx, start, K) == (L0, M0)          # the start render fits: no growth
    assert gpu_ctx.capacity() == (max(M0, 64), max(L0, 32))
    res = gpu_ctx.track_frame(0, start, K, tc, w)
    pc, bc = gpu_ctx.capacity()
    assert pc > M1 and bc > L1, (pc, bc, M1, L1)                 # grown from the loop's maxima
    assert list(res.pose.translation) == list(ref.pose.translation)
    assert list(res.pose.rotation_tangent) == list(ref.pose.rotation_tangent)
    assert res.final_loss == ref.final_loss and res.iterations_run == ref.iterations_run
    # API render and tracking_gradient: the same growth protocol, same results as with room to spare
    big = gpu_ctx.render(ref.pose, K)
    tg_ref = gpu_ctx.tracking_gradient(0, ref.pose, K, w)
    gpu_ctx.reserve(M0, L0)
    small = gpu_ctx.render(ref.pose, K)
    assert (small.per_pixel_count == big.per_pixel_count).all() and (small.color == big.color).all()
    gpu_ctx.reserve(M0, L0)
    tg = gpu_ctx.tracking_gradient(0, ref.pose, K, w)
    assert np.array_equal(tg[1], tg_ref[1])


def test_mapping_overflow_reported_then_matches(gpu_ctx, orc):
    """map_step with the binning capacities reserved below its views' lists: the mapping forward's
    lists are placed by one atomic each (k_tile_sort any_order, the last CTA recording M), so a
    list that does not fit must still raise the overflow — map_step reports it (EUnsupported: the
    map was already stepping, mapper.cpp has no rerun) instead of returning a map from truncated
    lists — and after a render at those poses has grown the capacities the same call reproduces
    the run that never overflowed, bit for bit."""
    from paper_2403_16095_b200.abi import defaults_mapper
    K = make_intrinsics(64, 48, 90.0)
    truth = _cluster_scene(orc)
    poses = [pose(), perturbed(pose(), [0.01, -0.02, 0.01, 0.03, -0.02, 0.01])]
    gpu_ctx.upload(to_api_map(truth))
    for s, p in enumerate(poses):
        r = gpu_ctx.render(p, K)
        gpu_ctx.frame_upload(s, r.color, r.alpha_depth, 64, 48)
    rng = np.random.default_rng(17)
    pert = f32_round(truth)
    pert.mean = (pert.mean + 0.01 * rng.standard_normal(pert.mean.shape)).astype(np.float32).astype(np.float64)
    mc = defaults_mapper()
    mc.densify_interval = 0
    gpu_ctx.upload(to_api_map(pert))
    exts = [_list_extent(gpu_ctx, p, K) for p in poses]
    L, M = max(e[0] for e in exts), max(e[1] for e in exts)
    t_ref = gpu_ctx.map_step([0, 1], poses, K, mc, 6)
    a = gpu_ctx.download()
    gpu_ctx.upload(to_api_map(pert))
    gpu_ctx.reserve(M // 3, max(L // 3, 32))
    with pytest.raises(NotImplementedError, match="pair capacity"):
        gpu_ctx.map_step([0, 1], poses, K, mc, 6)
    gpu_ctx.upload(to_api_map(pert))
    for p in poses:
        gpu_ctx.render(p, K)   # the render API grows the capacities to these views' lists
    pc, bc = gpu_ctx.capacity()
    assert pc >= M and bc >= L, (pc, bc, M, L)
    t = gpu_ctx.map_step([0, 1], poses, K, mc, 6)
    b = gpu_ctx.download()
    assert np.array_equal(t, t_ref)
    for k in ("mean", "log_scale", "quat", "opacity_logit", "sh"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k

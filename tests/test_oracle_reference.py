"""Pins the CPU oracle (oracle/gsf_oracle.cpp) to the reference's own tests.

Each test restates one reference test case (file:line cited) against the fp64 restatement, so a
transcription error in the oracle shows up here before it can mask a GPU bug.  CPU only.
"""
import math

import numpy as np
import pytest

from paper_2403_16095_b200.abi import (defaults_mapper, defaults_raster, defaults_tracker, defaults_weights)
from helpers import (axis_primitive, golden, make_intrinsics, one_pixel_camera, perturbed, pose, rotation_error,
                     scene, translation_error)


def test_two_primitive_pixel_kat(orc):
    """test_rasterizer.cpp:39-63"""
    g = golden("reference_kats.json")["two_primitive_pixel"]
    m = scene([axis_primitive(1.0, 0.6, [1, 0, 0]), axis_primitive(2.0, 0.8, [0, 1, 0])])
    K = one_pixel_camera()
    r = orc.render(m, pose(), K, np.array([[1.0]]))
    e = g["expect"]
    tol = 1e-12
    assert np.allclose(r.color[0, 0], e["color"], rtol=tol, atol=1e-14)
    assert r.opacity[0, 0] == pytest.approx(e["opacity"], rel=tol)
    assert r.alpha_depth[0, 0] == pytest.approx(e["alpha_depth"], rel=tol)
    assert r.median_valid[0, 0] == 1 and r.median_depth[0, 0] == pytest.approx(1.0)
    assert r.uncertainty[0, 0] == pytest.approx(e["uncertainty"], rel=tol)
    assert r.final_transmittance[0, 0] == pytest.approx(e["final_transmittance"], rel=tol)
    assert r.per_pixel_count[0, 0] == 2 and r.dominant[0, 0] == 0 and r.median_prim[0, 0] == 0
    rs, prim, alpha, tr = r.record()
    assert list(prim) == [0, 1] and tr[0] == pytest.approx(1.0) and tr[1] == pytest.approx(0.4, rel=tol)


def test_empty_frame(orc):
    """test_rasterizer.cpp:65-77"""
    m = scene([])
    r = orc.render(m, pose(), make_intrinsics(16, 12, 20.0))
    assert (r.opacity == 0).all() and (r.per_pixel_count == 0).all() and (r.final_transmittance == 1).all()
    assert not r.has_uncertainty


def test_non_finite_rejected_with_index(orc):
    """test_rasterizer.cpp:79-90"""
    m = orc.random_scene(3, 5)
    m.mean[3, 1] = float("nan")
    with pytest.raises(orc.OracleError) as ei:
        orc.render(m, pose(), make_intrinsics(8, 8, 10.0))
    assert "3" in str(ei.value) and "non-finite" in str(ei.value)


def test_tiled_matches_brute_force(orc):
    """test_rasterizer.cpp:119-134: 20 seeds x 200 primitives x 64^2 within 1e-5."""
    rng = np.random.default_rng(0)
    for seed in range(20):
        m = orc.random_scene(100 + seed, 200, 4 if seed % 3 == 0 else 1)
        K = make_intrinsics(64, 64, 60.0)
        obs = orc.wavy_depth(64, 64, 2.5)
        p = pose(0.03 * rng.standard_normal(3), 0.05 * rng.standard_normal(3))
        a = orc.render(m, p, K, obs)
        b = orc.render(m, p, K, obs, brute_force=True)
        d = max(np.abs(a.color - b.color).max(), np.abs(a.alpha_depth - b.alpha_depth).max(),
                np.abs(a.opacity - b.opacity).max(), np.abs(a.uncertainty - b.uncertainty).max())
        assert (a.median_valid == b.median_valid).all()
        d = max(d, np.abs(np.where(a.median_valid == 1, a.median_depth - b.median_depth, 0)).max())
        assert d < 1e-5


def test_blend_invariants(orc):
    """test_rasterizer.cpp:156-193"""
    cfg = defaults_raster()
    cfg.termination_threshold = 0.0
    for seed in range(6):
        m = orc.random_scene(300 + seed, 120, 1, 0.99)
        r = orc.render(m, pose(), make_intrinsics(48, 40, 45.0), cfg=cfg)
        o = r.opacity
        assert (o >= 0).all() and (o <= 1 + 1e-12).all()
        assert np.abs(o + r.final_transmittance - 1).max() < 1e-6
        assert (r.median_valid[r.per_pixel_count == 0] == 0).all()
        rs, prim, alpha, tr = r.record()
        for pi in range(48 * 40):
            prev, expect = 1.0, -1
            for e in range(rs[pi], rs[pi + 1]):
                assert tr[e] <= prev + 1e-15
                if expect < 0 and tr[e] >= 0.5 and tr[e] * (1 - alpha[e]) < 0.5:
                    expect = prim[e]
                prev = tr[e]
            assert r.median_prim.flat[pi] == expect


def test_uncertainty_absent_and_zero_at_holes(orc):
    """test_rasterizer.cpp:208-225"""
    m = orc.random_scene(88, 60)
    K = make_intrinsics(32, 32, 30.0)
    r = orc.render(m, pose(), K)
    assert not r.has_uncertainty and (r.uncertainty == 0).all()
    obs = np.full((32, 32), 2.0)
    obs[7, 5] = 0.0
    obs[3, 9] = 100.0
    r2 = orc.render(m, pose(), K, obs)
    assert r2.has_uncertainty and r2.uncertainty[7, 5] == 0 and r2.uncertainty[3, 9] == 0


def test_grazing_primitive_culled(orc):
    """test_rasterizer.cpp:227-255"""
    C0 = 0.28209479177387814
    wall = dict(mean=[0, 0, 3.0], scale=0.4, opacity=0.9, sh=[[0, 0, 0]])
    grazer = dict(mean=[1.8, -0.4, 0.12], scale=0.22, opacity=0.95, sh=[[(1 - 0.5) / C0, (0 - .5) / C0, (0 - .5) / C0]])
    K = make_intrinsics(32, 24, 30.0)
    clean = orc.render(scene([wall]), pose(), K)
    mixed = orc.render(scene([wall, grazer]), pose(), K)
    assert list(mixed.visible) == [1, 0]
    assert (clean.color == mixed.color).all() and (clean.opacity == mixed.opacity).all()
    assert clean.alpha_depth[12, 16] > 2.5


def test_screen_covariance_kat(orc):
    """test_geometry.cpp:160-172: isotropic sigma 0.1 at z=2, f=100 -> cov2d 25.3 (0.3 dilation)."""
    g = golden("reference_kats.json")["screen_covariance"]
    c = g["camera"]
    from paper_2403_16095_b200.abi import Intrinsics
    K = Intrinsics(c["fx"], c["fy"], c["cx"], c["cy"], c["width"], c["height"], 1.0, c["near"], c["far"])
    m = scene([dict(mean=[0, 0, 2.0], scale=0.1, opacity=0.5, color=[0.5, 0.5, 0.5])])
    cfg = defaults_raster()
    cfg.alpha_skip = 0.0
    r = orc.render(m, pose(), K, cfg=cfg)
    # the mean projects to (60, 40): a pixel center at dx = k + 0.5 has alpha = 0.5 exp(-dx^2 / (2 * 25.3))
    for k in range(0, 12):
        dx = k + 0.5
        assert r.opacity[39, 60 + k] == pytest.approx(0.5 * math.exp(-0.5 * (dx * dx + 0.25) / g["expect_cov2d"]), rel=1e-9)


def _linear_probe(rng, w, h, with_unc):
    """test_gradients.cpp:17-37"""
    a_color = rng.standard_normal((h, w, 3))
    a_depth = rng.standard_normal((h, w))
    a_op = rng.standard_normal((h, w))
    a_unc = rng.standard_normal((h, w)) if with_unc else None
    a_med = rng.standard_normal((h, w))
    return a_color, a_depth, a_op, a_unc, a_med


def test_gradients_match_finite_differences(orc):
    """test_gradients.cpp:85-105 (seeds/structure restated with numpy draws)."""
    from paper_2403_16095_b200.abi import defaults_raster
    checked = skipped = 0
    for seed in range(8):
        rng = np.random.default_rng(1000 + seed)
        n = 4 if seed < 3 else (12 if seed < 6 else 30)
        K_sh = 4 if seed % 3 == 1 else (16 if seed == 7 else 1)
        m = orc.random_scene(1000 + seed, n, K_sh)
        K = make_intrinsics(24, 24, 24 * 0.9)
        cfg = defaults_raster()
        cfg.alpha_skip, cfg.termination_threshold, cfg.footprint_sigma = 0.0, 0.0, 8.0   # gradcheck.cpp:21-27
        obs = orc.wavy_depth(24, 24, 2.5) if seed % 2 == 0 else None
        p = pose(0.02 * rng.standard_normal(3), 0.03 * rng.standard_normal(3))
        probe = _linear_probe(rng, 24, 24, obs is not None)
        rep = orc.gradcheck_linear(m, p, K, cfg, obs, *probe)
        assert rep.max_rel_err < 1e-5, (seed, rep.worst_index, rep.worst_analytic, rep.worst_fd)
        checked += rep.checked
        skipped += rep.skipped
    assert checked > 500 and skipped < 0.05 * (checked + skipped)


def test_zero_upstream_zero_bundle(orc):
    """test_gradients.cpp:107-122"""
    m = orc.random_scene(7, 10)
    K = make_intrinsics(16, 16, 15.0)
    r = orc.render(m, pose(), K)
    g = orc.render_backward(m, pose(), K, r)
    assert np.all(g.d_pose == 0) and np.all(g.d_mean == 0) and np.all(g.d_quat == 0)


def test_symmetric_scene_zero_lateral_pose_gradient(orc):
    """test_gradients.cpp:164-179"""
    m = scene([dict(mean=[0, 0, 2.0], scale=0.08, opacity=0.7, sh=[[0.3, 0.1, -0.2]])])
    K = make_intrinsics(33, 33, 30.0)
    r = orc.render(m, pose(), K)
    g = orc.render_backward(m, pose(), K, r, d_opacity=np.ones((33, 33)))
    assert abs(g.d_pose[3]) < 1e-10 and abs(g.d_pose[4]) < 1e-10


def test_mapping_loss_kat(orc):
    """test_losses.cpp:169-198"""
    e = golden("reference_kats.json")["mapping_loss_single_pixel"]["expect"]
    m = scene([axis_primitive(1.0, 0.6, [1, 0, 0]), axis_primitive(2.0, 0.8, [0, 1, 0])])
    K = one_pixel_camera()
    obs = np.array([[1.0]])
    r = orc.render(m, pose(), K, obs)
    out, (dc, dad, dmd, du, dls) = orc.mapping_loss(m, r, r.color.copy(), obs, K, defaults_weights())
    assert out.color == pytest.approx(0.0) and out.ssim == pytest.approx(0.0, abs=1e-12)
    assert out.geo == pytest.approx(e["geo"], rel=1e-12) and out.align == pytest.approx(e["align"], rel=1e-12)
    assert out.var == pytest.approx(e["var"], rel=1e-12) and out.total == pytest.approx(e["total"], rel=1e-12)
    assert dad[0] == pytest.approx(e["d_alpha_depth"]) and dmd[0] == pytest.approx(e["d_median_depth"])
    assert du[0] == pytest.approx(e["d_uncertainty"]) and np.abs(dc).max() < 1e-12 and (dls == 0).all()


def test_tracking_loss_zero_at_perfect_frame(orc):
    """test_losses.cpp:235-259"""
    m = orc.random_scene(41, 25, 1, 0.98)
    K = make_intrinsics(32, 24, 30.0)
    r = orc.render(m, pose(), K)
    out, dc, dd = orc.tracking_loss(r, r.color, r.alpha_depth, K, defaults_weights())
    assert out.total == 0.0 and out.valid_color > 0 and (dc == 0).all() and (dd == 0).all()


def test_ssim_hand_cases_and_gradient(orc):
    """test_losses.cpp:100-149"""
    rng = np.random.default_rng(11)
    x = rng.random((16, 20, 3))
    assert 1 - orc.ssim(x, x, 20, 16) == pytest.approx(0.0, abs=1e-14)
    c1 = 1e-4
    assert 1 - orc.ssim(np.zeros((16, 16, 3)), np.ones((16, 16, 3)), 16, 16) == pytest.approx(1 - c1 / (1 + c1), rel=1e-12)
    assert 1 - orc.ssim(np.zeros((3, 4, 3)), np.ones((3, 4, 3)), 4, 3) == pytest.approx(1 - c1 / (1 + c1), rel=1e-12)
    for (w, h) in ((16, 13), (7, 5)):
        x = rng.random((h, w, 3))
        y = rng.random((h, w, 3))
        _, g = orc.ssim(x, y, w, h, gradient=True)
        for _ in range(20):
            i = rng.integers(0, w * h * 3)
            xp, xm = x.copy().ravel(), x.copy().ravel()
            xp[i] += 1e-5
            xm[i] -= 1e-5
            fd = (orc.ssim(xp, y, w, h) - orc.ssim(xm, y, w, h)) / 2e-5
            assert g[i] == pytest.approx(fd, rel=1e-5, abs=1e-9)


def test_uncertainty_kats(orc):
    """test_map.cpp:118-155 (the hand-built records are produced by a 1-pixel render)."""
    K = one_pixel_camera()
    m = scene([dict(mean=[0, 0, 1.5], scale=0.05, opacity=0.9, color=[0.5, 0.5, 0.5])])
    ra = orc.render(m, pose(), K)
    n = orc.accumulate_uncertainty(m, [ra], [np.array([[2.0]])], [pose()], K)
    assert n == 1 and m.observed[0] == 1 and m.uncertainty[0] == pytest.approx(0.225, rel=1e-12)
    mb = scene([dict(mean=[0, 0, 1.5], scale=0.05, opacity=0.5, color=[0.5, 0.5, 0.5])])
    rb = orc.render(mb, pose(), K)
    m2 = scene([dict(mean=[0, 0, 1.5], scale=0.05, opacity=0.9, color=[0.5, 0.5, 0.5])])
    orc.accumulate_uncertainty(m2, [ra, rb], [np.array([[2.0]]), np.array([[1.6]])], [pose(), pose()], K)
    assert m2.uncertainty[0] == pytest.approx(0.115, rel=1e-12)


def test_prune_kat(orc):
    """test_map.cpp:189-211"""
    m = scene([dict(mean=[0, 0, 2], scale=0.1, opacity=0.8)] * 3)
    m.uncertainty[:] = [0.225, 0.0, 0.024]
    assert orc.prune_unreliable(m) == 1
    assert 1 / (1 + math.exp(-m.opacity_logit[0])) == pytest.approx(0.005, rel=1e-12)
    assert orc.prune_unreliable(m) == 0


def test_adam_first_step(orc):
    """test_map.cpp:64-73"""
    import ctypes as C
    x = np.array([1.0, -2.0])
    g = np.array([3.0, -0.004])
    mm, vv = np.zeros(2), np.zeros(2)
    t = C.c_uint64(0)
    dp = C.POINTER(C.c_double)
    orc.lib().orc_adam_step(x.ctypes.data_as(dp), g.ctypes.data_as(dp), mm.ctypes.data_as(dp), vv.ctypes.data_as(dp),
                            2, C.byref(t), 0.1, 0.9, 0.999, 1e-8)
    assert x[0] == pytest.approx(0.9, rel=1e-6) and x[1] == pytest.approx(-1.9, rel=1e-3) and t.value == 1


def test_tracking_stationary_and_recovers(orc):
    """test_tracker.cpp:192-244"""
    K = make_intrinsics(48, 36, 40.0)
    m = orc.random_scene(7, 60)
    r = orc.render(m, pose(), K)
    tc = defaults_tracker()
    tc.iterations = 10
    res = orc.track_frame(m, r.color, r.alpha_depth, pose(), K, tc, defaults_weights(True), defaults_raster())
    assert np.linalg.norm(list(res.pose.rotation_tangent)) <= 1e-15 and res.final_loss == 0.0
    assert not res.degraded and res.iterations_run == 10
    K = make_intrinsics(64, 48, 55.0)
    m = orc.random_scene(19, 80)
    r = orc.render(m, pose(), K)
    start = perturbed(pose(), [0.004, -0.003, 0.002, 0.008, -0.006, 0.004])
    tc.iterations = 40
    res = orc.track_frame(m, r.color, r.alpha_depth, start, K, tc, defaults_weights(True), defaults_raster())
    assert rotation_error(res.pose, pose()) < 0.35 * rotation_error(start, pose())
    assert translation_error(res.pose, pose()) < 0.35 * translation_error(start, pose())
    again = orc.track_frame(m, r.color, r.alpha_depth, start, K, tc, defaults_weights(True), defaults_raster())
    assert list(again.pose.translation) == list(res.pose.translation) and again.final_loss == res.final_loss


def test_tracking_empty_view_degraded(orc):
    """test_tracker.cpp:246-263"""
    m = orc.random_scene(3, 30)
    K = make_intrinsics(32, 24, 28.0)
    away = pose((math.pi, 0, 0))
    res = orc.track_frame(m, np.full((24, 32, 3), 0.5), orc.wavy_depth(32, 24, 2.0), away, K, defaults_tracker(),
                          defaults_weights(True), defaults_raster())
    assert res.degraded and res.iterations_run == 0


def test_ba_noop_at_optimum(orc):
    """test_tracker.cpp:319-363"""
    m = orc.random_scene(31, 50)
    K = make_intrinsics(48, 36, 40.0)
    mc = defaults_mapper()
    mc.weights.w_ssim = mc.weights.w_align = mc.weights.w_iso = mc.weights.w_var = 0.0
    poses = [pose(), perturbed(pose(), [0.02, -0.01, 0.03, 0.05, 0.02, -0.04]),
             perturbed(pose(), [-0.03, 0.02, -0.01, -0.04, 0.03, 0.05])]
    frames = []
    for p in poses:
        r = orc.render(m, p, K)
        frames.append((r.color.copy(), r.alpha_depth.copy()))
    st = orc.MapState(m, mc)
    trace, out_poses = st.sliding_ba(frames, poses, [0, 10, 20], K, defaults_tracker(), mc, 5)
    assert (trace == 0).all()
    m2 = st.get()
    assert (m2.mean == m.mean).all() and (m2.opacity_logit == m.opacity_logit).all()


def test_map_step_reduces_loss(orc):
    """test_map.cpp:391-423"""
    K = make_intrinsics(48, 36, 40.0)
    truth = orc.random_scene(83, 40, 1, 0.95, 0.05, 0.2)
    gt = orc.render(truth, pose(), K)
    obs = np.where(gt.opacity > 0.5, gt.alpha_depth, 0.0)
    rng = np.random.default_rng(83)
    pert = truth
    pert.mean = pert.mean + 0.02 * rng.standard_normal(pert.mean.shape)
    pert.sh[:, 0] = pert.sh[:, 0] + 0.15 * rng.standard_normal((40, 3))
    mc = defaults_mapper()
    mc.densify_interval = 0
    st = orc.MapState(pert, mc)
    trace = st.map_step([(gt.color.copy(), obs)], [pose()], K, mc, 60)
    assert trace[-1] < 0.7 * trace[0]


def _tiny_camera(w, h):
    """test_map.cpp:17-27"""
    from paper_2403_16095_b200 import api
    return api.intrinsics(10.0, 10.0, 0.5 * w, 0.5 * h, w, h, near_plane=0.1, far_plane=100.0)


def test_backproject_initialize_kats(orc):
    """test_map.cpp:246-283 (initialize_map): stride sampling, footprint scale, colour decode, axis pixel."""
    from paper_2403_16095_b200.abi import defaults_mapper
    mc = defaults_mapper()
    K = _tiny_camera(4, 4)
    rgb = np.tile(np.array([0.2, 0.4, 0.6]), (4, 4, 1))
    depth = np.full((4, 4), 2.0)
    assert orc.backproject(rgb, depth, pose(), K, mc, 1).mean.shape[0] == 16
    half = orc.backproject(rgb, depth, pose(), K, mc, 2)
    assert half.mean.shape[0] == 4
    assert half.log_scale[0, 0] == pytest.approx(math.log((2.0 / 10.0) * 2 * 0.5))
    assert half.sh[0, 0, 0] * 0.28209479177387814 + 0.5 == pytest.approx(0.2, rel=1e-12)
    assert 1.0 / (1.0 + math.exp(-half.opacity_logit[0])) == pytest.approx(0.5)
    K3 = _tiny_camera(3, 3)
    d3 = np.zeros((3, 3))
    d3[1, 1] = 2.0
    one = orc.backproject(np.full((3, 3, 3), 0.5), d3, pose(), K3, mc, 1)
    assert one.mean.shape[0] == 1 and np.linalg.norm(one.mean[0] - [0, 0, 2]) < 1e-12
    assert orc.backproject(np.full((3, 3, 3), 0.5), np.zeros((3, 3)), pose(), K3, mc, 1).mean.shape[0] == 0


def test_backproject_spawn_kats(orc):
    """test_map.cpp:285-315 (spawn_gaussians): thin pixels with valid depth only."""
    from paper_2403_16095_b200.abi import defaults_mapper
    mc = defaults_mapper()
    K = _tiny_camera(4, 3)
    rgb = np.full((3, 4, 3), 0.3)
    depth = np.full((3, 4), 1.5)
    assert orc.backproject(rgb, depth, pose(), K, mc, 1, opacity=np.ones((3, 4))).mean.shape[0] == 0
    depth[1, 2] = 0.0
    spawned = orc.backproject(rgb, depth, pose(), K, mc, 1, opacity=np.zeros((3, 4)))
    assert spawned.mean.shape[0] == 11 and np.allclose(spawned.mean[:, 2], 1.5)
    partial = np.full((3, 4), 0.8)
    partial[1, 1] = 0.4
    assert orc.backproject(rgb, np.full((3, 4), 1.5), pose(), K, mc, 1, opacity=partial).mean.shape[0] == 1


def _plane_map(orc, specs):
    """test_map.cpp:44-51 plane_primitive(x, y, z, scale, opacity)."""
    from helpers import logit
    m = orc.empty_map(len(specs), 1)
    for i, (x, y, z, sc, op) in enumerate(specs):
        m.mean[i] = [x, y, z]
        m.log_scale[i] = math.log(sc)
        m.opacity_logit[i] = logit(op)
    return m


def test_densify_kat(orc):
    """test_map.cpp:317-350: split large, clone small, cull faded, order of survivors."""
    from paper_2403_16095_b200.abi import defaults_mapper
    mc = defaults_mapper()
    mc.scene_extent = 4.0
    m = _plane_map(orc, [(0, 0, 2, 0.10, 0.9), (1, 0, 2, 0.01, 0.9), (0, 1, 2, 0.02, 1e-4), (1, 1, 2, 0.02, 0.9)])
    st = orc.MapState(m, mc)
    st.set_stats([1.0, 1.0, 0.0, 0.0], [1, 1, 0, 1])
    assert st.densify(mc) == (1, 1, 1)
    g = st.get()
    assert g.mean.shape[0] == 5
    assert g.mean[0, 0] == pytest.approx(1.0) and g.mean[1, 1] == pytest.approx(1.0)
    assert math.exp(g.log_scale[2, 0]) == pytest.approx(0.10 / 1.6, rel=1e-12)
    assert g.mean[4, 0] == pytest.approx(1.0)
    assert st.densify(mc) == (0, 0, 0) and st.get().mean.shape[0] == 5


def test_per_primitive_rho_bounds_are_safe(orc):
    """blend_rho_bounds (gsf_shared.cuh): the per-primitive band around the footprint cutoff
    (rasterizer.cpp:110) must contain every fp32-vs-fp64 rho difference, so that a fast-path pair is
    an fp64 contribution and a pair above rho_hi an fp64 skip.  4,000 random primitives (means up to
    6,000 px off-image, screen sigmas 0.3-300 px, conditioning to 1e-4), every pixel of their boxes."""
    import ctypes as C
    lib = orc.lib()
    lib.mir_band_check.argtypes = [C.c_int, C.c_uint64, C.c_void_p]
    for seed in (0, 1):
        out = np.zeros(5)
        assert lib.mir_band_check(2000, seed, out.ctypes.data) == 0
        violations, worst, tested, guarded, worst_capped = out
        assert violations == 0 and tested > 1e8
        assert worst < 0.25        # the bound carries a factor 4 on top of its own worst case
        assert worst_capped < 1.0  # means far off the image fall back to the global band
        assert guarded < 1e-4 * tested
